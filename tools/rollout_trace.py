#!/usr/bin/env python3
"""Phase timing inside the fused rollout kernel (CTA 0, globaltimer stamps written when
GMI_ROLLOUT_TRACE=1). Development aid: prints per-phase microseconds averaged over steps."""
import os
import sys

os.environ["GMI_ROLLOUT_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

from paper_2206_08482_b200.ppo import PpoConfig, Trainer  # noqa: E402


def main():
    path = sys.argv[1] if len(sys.argv) > 1 else os.path.join(os.path.dirname(__file__), "..", "configs",
                                                               "at_4096env_3x256.cfg")
    cfg = PpoConfig.from_config_file(path)
    cfg.gmis_per_gpu, cfg.gmi_backend, cfg.sm_per_gmi = 1, 0, 0  # one GMI on the whole GPU
    t = Trainer(cfg)
    for _ in range(3):  # the hook's rollout is consumed by the next iteration
        t.rollout()
        t.iteration()
    t.rollout()
    tr = t.get("rollout_trace").view(np.int64).reshape(cfg.horizon, 16).astype(np.float64)
    L = len(cfg.hidden)
    names, cols = [], []
    prev = None
    order = [(2 * l, f"L{l} mma->acc") for l in range(L)]
    seq = []
    for l in range(L):
        seq += [(2 * l, f"wait acc L{l}"), (2 * l + 1, f"epilogue L{l}")]
    seq += [(10, "wait acc head"), (11, "head+actions"), (12, "dynamics"), (13, "obs write")]
    print(f"steps {cfg.horizon}, total {(tr[-1, 12] - tr[0, 0]) / 1e3:.1f} us (step 0 acc0 -> last dynamics)")
    for s in range(1, cfg.horizon):
        pass
    rows = []
    for i, (k, name) in enumerate(seq):
        pk = seq[i - 1][0] if i > 0 else 13
        d = tr[:, k] - (tr[:, pk] if i > 0 else np.roll(tr[:, 13], 1))
        rows.append((name, np.median(d[1:]) / 1e3))
    for name, us in rows:
        print(f"{name:16s} {us:8.2f} us")
    print(f"per step         {np.median(np.diff(tr[:, 0])) / 1e3:8.2f} us")


if __name__ == "__main__":
    main()
