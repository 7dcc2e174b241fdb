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
    ap.add_argument("--split", type=int, default=0, help="AsyncDecoupled across ranks (decoupled = 2)")
    ap.add_argument("--backend", type=int, default=-1, help="gmi_backend (default: 1 if decoupled else 0)")
    ap.add_argument("--out")
    a = ap.parse_args()
    import torch.distributed as dist
    from paper_2206_08482_b200.ppo import PpoConfig, Trainer

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(a.port))
    dist.init_process_group("gloo", rank=a.rank, world_size=a.world)
    if a.split:
        return split_rank(a, dist, PpoConfig, Trainer)
    t = Trainer(PpoConfig(obs_dim=12, act_dim=3, hidden=[64, 64], num_envs=a.envs, num_gpus=a.world, rank=a.rank,
                          gmis_per_gpu=a.gmis, comm=1, device=0, decoupled=a.decoupled,
                          gmi_backend=a.backend if a.backend >= 0 else (1 if a.decoupled else 0)))
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


def split_rank(a, dist, PpoConfig, Trainer):
    """AsyncDecoupled across ranks: [0, G/2) serve, G/2 + s trains on serving rank s's envs;
    each pair wired with the link handles (gmi_ppo_link_handle -> gloo -> gmi_ppo_link_attach)."""
    t = Trainer(PpoConfig(obs_dim=12, act_dim=3, hidden=[64, 64], num_envs=a.envs, num_gpus=a.world, rank=a.rank,
                          comm=1, device=0, decoupled=2))
    handles = [None] * a.world
    dist.all_gather_object(handles, t.link_handle())
    t.link_attach(handles[(a.rank + a.world // 2) % a.world])
    serving = a.rank < a.world // 2
    # the trainer ranks' own data-parallel job: peer exchange among them, in trainer-rank order
    comm = [None] * a.world
    dist.all_gather_object(comm, None if serving or a.world == 2 else t.comm_handle())
    if not serving and a.world > 2:
        t.comm_attach(comm[a.world // 2:])
    dist.barrier()
    steps = [t.iteration().env_steps for _ in range(a.iters)]
    dist.barrier()  # the trainer's last snapshot push has landed in the serving rank's window
    out = {"params": t.get("params"), "steps": np.array(steps)}
    fields = ("done", "rew", "act", "logp", "adv", "obs") if serving else ("trained_logp", "act", "adv", "obs")
    for f in fields:
        out[f] = t.get(f)
    np.savez(a.out, **out)
    dist.barrier()
    t.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
