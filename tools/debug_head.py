#!/usr/bin/env python3
"""Development check: fused vs per-kernel PPO head on the same minibatch, repeated, with
allocation noise in between (uninitialised-memory / race detector)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from golden_util import param_layout  # noqa: E402
from paper_2206_08482_b200.ppo import PpoConfig, Trainer  # noqa: E402


def grads(unfused, S, A, hidden, envs):
    if unfused:
        os.environ["GMI_HEAD_UNFUSED"] = "1"
    else:
        os.environ.pop("GMI_HEAD_UNFUSED", None)
    t = Trainer(PpoConfig(obs_dim=S, act_dim=A, hidden=hidden, num_envs=envs))
    B = envs * 32 // 4
    rng = np.random.default_rng(S)
    X = rng.uniform(-1, 1, (B, S)).astype(np.float32)
    act = rng.standard_normal((B, A)).astype(np.float32)
    oldlp = (rng.standard_normal(B) - 3).astype(np.float32)
    adv = rng.standard_normal(B).astype(np.float32)
    ret = rng.standard_normal(B).astype(np.float32)
    g = t.minibatch_grad(X, act, oldlp, adv, ret)
    t.close()
    return g


def main():
    S, A, hidden, envs = 60, 8, [256, 256, 256], 64
    lay = param_layout(S, A, hidden)
    ref = grads(True, S, A, hidden, envs)
    for trial in range(4):
        junk = torch.randn(1 << 26, device="cuda") * (trial + 1)  # dirty the allocator
        g = grads(False, S, A, hidden, envs)
        del junk
        worst = []
        for key, t in lay.items():
            if not isinstance(key, tuple):
                continue
            for part, n in (("w", t["out_p"] * t["in_p"]), ("b", t["out_p"])):
                a, b = g[t[part]:t[part] + n], ref[t[part]:t[part] + n]
                rel = np.linalg.norm(a - b) / (np.linalg.norm(b) + 1e-20)
                worst.append((rel, key, part, np.linalg.norm(b)))
        worst.sort(reverse=True)
        print(trial, [(f"{r:.2e}", k, p, f"{nb:.2e}") for r, k, p, nb in worst[:4]], flush=True)


if __name__ == "__main__":
    main()
