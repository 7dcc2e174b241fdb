import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2206_08482_b200.ppo import PpoConfig, Trainer
cfg = dict(obs_dim=12, act_dim=3, hidden=[64, 64], num_envs=64)
a = Trainer(PpoConfig(**cfg)); a.iteration(); pa = a.get("params"); ma = a.get("adam_m")
os.environ["GMI_ADAM_FUSED"] = "1"
b = Trainer(PpoConfig(**cfg)); b.iteration(); pb = b.get("params"); mb = b.get("adam_m")
d = np.abs(pa - pb); print("params max", d.max(), "n diff", (d > 0).sum(), "of", d.size)
print("m max", np.abs(ma - mb).max())
idx = np.nonzero(d)[0][:20]; print(idx)
