#!/usr/bin/env python3
"""Per-tile timeline of one GEMM launch (CTA 0): GMI_GEMM_TRACE=<phase id> stamps the last
launch of that phase in an iteration. Development aid; needs a trace build: make -C paper_2206_08482_b200/csrc clean all TRACE=1.
    python tools/gemm_trace.py 7     # training forward GEMMs (last = layer L-1)"""
import os
import sys

phase = sys.argv[1] if len(sys.argv) > 1 else "7"
os.environ["GMI_GEMM_TRACE"] = phase
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

from paper_2206_08482_b200.ppo import PpoConfig, Trainer  # noqa: E402

NAMES = {0: "mma tile start", 1: "acc free", 2: "first stage", 3: "mma committed", 4: "epi acc ready",
         5: "epi chunk0 stored", 9: "epi chunk1 stored", 6: "epi done", 7: "tma tile start", 8: "tma tile issued"}


def main():
    cfg = PpoConfig.from_config_file(os.path.join(os.path.dirname(__file__), "..", "configs", "at_4096env_3x256.cfg"))
    t = Trainer(cfg)
    for _ in range(3):
        t.iteration()
    tr = t.get("gemm_trace").view(np.int64).reshape(8, 16).astype(np.float64)
    t0 = tr[0, 7] if tr[0, 7] > 0 else tr[0, 0]
    for lt in range(8):
        if tr[lt].max() <= 0:
            break
        row = sorted((tr[lt, k] - t0, n) for k, n in NAMES.items() if tr[lt, k] > 0)
        print(f"tile {lt}: " + ", ".join(f"{n} {v / 1e3:.2f}" for v, n in row))


if __name__ == "__main__":
    main()
