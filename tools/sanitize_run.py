#!/usr/bin/env python3
"""Small PPO iterations for compute-sanitizer (memcheck / racecheck / synccheck / initcheck):
the SMALL 12:64:64:3 shape with 2 GMIs (per-layer GEMMs, fused rollout / head, K1 fold), the
3x256 bench shape at 128 envs (cluster rollout, weight-stationary GEMMs, fused head), and the
single-rank peer exchange. Two iterations each: eager, then the CUDA-graph replay.

    compute-sanitizer --tool memcheck python tools/sanitize_run.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2206_08482_b200.ppo import PpoConfig, Trainer  # noqa: E402

which = sys.argv[1:] or ["small", "at", "xchg"]
cases = {
    "small": PpoConfig(obs_dim=12, act_dim=3, hidden=[64, 64], num_envs=64, gmis_per_gpu=2),
    "at": PpoConfig(obs_dim=60, act_dim=8, hidden=[256, 256, 256], num_envs=128),
    "xchg": PpoConfig(obs_dim=12, act_dim=3, hidden=[64, 64], num_envs=64, comm=1),
}
for name in which:
    t = Trainer(cases[name])
    for _ in range(2):
        s = t.iteration()
    print(name, "ok", s.policy_loss, flush=True)
    t.close()
