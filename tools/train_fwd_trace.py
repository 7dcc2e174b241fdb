#!/usr/bin/env python3
"""Phase timing inside the fused training-forward kernel (CTA 0, globaltimer stamps written
when GMI_TRAIN_FWD_TRACE=1 and GMI_TRAIN_FWD=1). Development aid; needs a trace build: make -C paper_2206_08482_b200/csrc clean all TRACE=1."""
import os
import sys

os.environ["GMI_TRAIN_FWD"] = "1"
os.environ["GMI_TRAIN_FWD_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

from paper_2206_08482_b200.ppo import PpoConfig, Trainer  # noqa: E402

NAMES = {0: "tile start", 1: "acc L0", 2: "acc L1", 3: "acc L2", 4: "epi L0 done", 5: "epi L1 done",
         6: "epi L2 done", 7: "acc head", 8: "G ready", 9: "acc MMA2/3", 10: "dact done", 11: "MMA L0 issue",
         12: "MMA2 issue"}


def main():
    cfg = PpoConfig.from_config_file(os.path.join(os.path.dirname(__file__), "..", "configs", "at_4096env_3x256.cfg"))
    t = Trainer(cfg)
    for _ in range(3):
        t.iteration()
    tr = t.get("train_fwd_trace").view(np.int64).reshape(4, 16).astype(np.float64)
    t0 = tr[0, 0]
    for ti in range(4):
        row = sorted((tr[ti, k] - t0, NAMES[k]) for k in NAMES if tr[ti, k] > 0)
        print(f"tile {ti}: " + ", ".join(f"{n} {v / 1e3:.2f}" for v, n in row))


if __name__ == "__main__":
    main()
