"""One rank of a multi-rank PPO job for tests/test_multirank_gpu.py: wires the peer exchange
over CUDA IPC (handles gathered with torch.distributed on gloo), runs `iters` iterations and
dumps the state the test compares. Every rank may sit on the same GPU (one process each)."""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rank", type=int)
    ap.add_argument("--world", type=int)
    ap.add_argument("--port", type=int)
    ap.add_argument("--envs", type=int)
    ap.add_argument("--gmis", type=int, default=1)
    ap.add_argument("--iters", type=int, default=2)
    ap.add_argument("--decoupled", type=int, default=0)
    ap.add_argument("--out")
    a = ap.parse_args()
    import torch.distributed as dist
    from paper_2206_08482_b200.ppo import PpoConfig, Trainer

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(a.port))
    dist.init_process_group("gloo", rank=a.rank, world_size=a.world)
    t = Trainer(PpoConfig(obs_dim=12, act_dim=3, hidden=[64, 64], num_envs=a.envs, num_gpus=a.world, rank=a.rank,
                          gmis_per_gpu=a.gmis, comm=1, device=0, decoupled=a.decoupled,
                          gmi_backend=1 if a.decoupled else 0))
    handles = [None] * a.world
    dist.all_gather_object(handles, t.comm_handle())
    t.comm_attach(handles)
    dist.barrier()
    for _ in range(a.iters):
        t.iteration()
    out = {"params": t.get("params")}
    for c in range(a.gmis):
        for f in ("done", "ep_count", "ep_step", "rew", "act"):
            out[f"{f}{c}"] = t.get(f, c)
    np.savez(a.out, **out)
    dist.barrier()
    t.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
