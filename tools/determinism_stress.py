#!/usr/bin/env python3
"""Repeat-run determinism check (development aid): pairs of identically configured trainers run
the same iterations and must end with bit-identical parameters; reports mismatches per mode.

    python tools/determinism_stress.py --reps 10 --envs 4096
"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--envs", type=int, default=4096)
    ap.add_argument("--iters", type=int, default=2)
    ap.add_argument("--modes", default="chain,plain")
    a = ap.parse_args()
    from paper_2206_08482_b200.ppo import PpoConfig, Trainer
    cfg = dict(obs_dim=60, act_dim=8, hidden=[256, 256, 256], num_envs=a.envs)
    for mode in a.modes.split(","):
        os.environ["GMI_FWD_CHAIN"] = "0" if mode == "plain" else "1"
        ref = Trainer(PpoConfig(**cfg))
        for _ in range(a.iters):
            ref.iteration()
        p0 = ref.get("params").view(np.uint32).copy()
        del ref
        bad = 0
        for r in range(a.reps):
            t = Trainer(PpoConfig(**cfg))
            for _ in range(a.iters):
                t.iteration()
            p = t.get("params").view(np.uint32)
            if not np.array_equal(p, p0):
                bad += 1
                d = np.nonzero(p != p0)[0]
                print(f"{mode} rep {r}: {d.size} params differ, first {d[:8].tolist()}", flush=True)
            del t
        print(f"{mode}: {bad} / {a.reps} runs differ from the first", flush=True)


if __name__ == "__main__":
    main()
