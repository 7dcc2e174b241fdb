#!/usr/bin/env python3
"""Per-tile timeline of the fused head kernel (CTA 0). Development aid; needs a trace build:
make -C paper_2206_08482_b200/csrc clean all TRACE=1."""
import os
import sys

os.environ["GMI_HEAD_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

from paper_2206_08482_b200.ppo import PpoConfig, Trainer  # noqa: E402

NAMES = {0: "mma: wait H", 1: "H landed", 2: "mma1 committed", 3: "G ready (mma)", 4: "mma2/3 committed",
         5: "loss: acc1 ready", 6: "loss: G written", 7: "dact: acc2 ready", 8: "dact: done"}


def main():
    path = sys.argv[1] if len(sys.argv) > 1 else os.path.join(os.path.dirname(__file__), "..", "configs",
                                                               "at_4096env_3x256.cfg")
    cfg = PpoConfig.from_config_file(path)
    cfg.gmis_per_gpu, cfg.gmi_backend, cfg.sm_per_gmi = 1, 0, 0  # one GMI on the whole GPU
    t = Trainer(cfg)
    for _ in range(3):
        t.iteration()
    tr = t.get("head_trace").view(np.int64).reshape(4, 16).astype(np.float64)
    t0 = tr[0, 0]
    for it in range(4):
        row = sorted((tr[it, k] - t0, n) for k, n in NAMES.items() if tr[it, k] > 0)
        print(f"tile {it}: " + ", ".join(f"{n} {v / 1e3:.2f}" for v, n in row))


if __name__ == "__main__":
    main()
