"""Debug aid: fused training forward (train_fwd.cu) vs the per-layer path, intermediate buffers."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2206_08482_b200.ppo import PpoConfig, Trainer

S, A, hidden, envs = 60, 8, [256, 256, 256], int(sys.argv[1]) if len(sys.argv) > 1 else 1000
cfg = dict(obs_dim=S, act_dim=A, hidden=hidden, num_envs=envs)
os.environ["GMI_TRAIN_FWD"] = "1"
fused = Trainer(PpoConfig(**cfg))
del os.environ["GMI_TRAIN_FWD"]
plain = Trainer(PpoConfig(**cfg))
B = envs * 32 // 4
rng = np.random.default_rng(S + A)
X = rng.uniform(-1, 1, (B, S)).astype(np.float32)
act = rng.standard_normal((B, A)).astype(np.float32)
oldlp = (rng.standard_normal(B) - 3).astype(np.float32)
adv = rng.standard_normal(B).astype(np.float32)
ret = rng.standard_normal(B).astype(np.float32)
g1 = fused.minibatch_grad(X, act, oldlp, adv, ret)
g2 = plain.minibatch_grad(X, act, oldlp, adv, ret)
for name in ["H00", "H01", "H10", "H11", "D02", "D12", "D01", "D00"]:
    a, b = fused.get(name).reshape(B, -1), plain.get(name).reshape(B, -1)
    d = np.abs(a - b)
    bad = np.argwhere(d > 1e-2 * (np.abs(b) + 1e-3))
    print(name, "max|d|", d.max(), "nbad", len(bad), "first", bad[:4].tolist(), "rows bad", np.unique(bad[:, 0])[:10].tolist() if len(bad) else [])
hp = fused.get("head_part"), plain.get("head_part")
print("head_part", np.abs(hp[0][:40] - hp[1][:40]).max(), hp[0][:20], hp[1][:20])
