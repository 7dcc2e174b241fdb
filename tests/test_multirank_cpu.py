"""World-size-2 data-parallel decomposition on CPU (gloo), using the CPU restatement.

Each rank plays one GPU of a 2-GPU x 1-GMI job (BASELINE config 2 layout, scaled down):
it owns the environments of its GMI ([N*c/n, N*(c+1)/n), reduction.hpp:164-166), computes
its minibatch gradient, and the ranks sum gradients with a gloo all-reduce -- the data path's
only collective. The result must equal the in-process sum over both GMIs, and every rank must
end with bit-identical parameters after the shared Adam step. Also checks that the
reference arm of bench.py runs under torchrun on rank 0 only.
"""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CFG = dict(obs_dim=12, act_dim=3, hidden=[32, 32], num_envs=64)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _minibatch_inputs(orc, gmi):
    N = CFG["num_envs"] // 2
    T = 32
    Bm = N * T // 4
    S, A = CFG["obs_dim"], CFG["act_dim"]
    obs = orc.get("obs", gmi).reshape(T + 1, N, S)[:T].reshape(T * N, S)[:Bm]
    act = orc.get("act", gmi).reshape(T * N, A)[:Bm]
    logp = orc.get("logp", gmi)[:Bm]
    adv = orc.get("adv", gmi)[:Bm]
    ret = orc.get("ret", gmi)[:Bm]
    adv = (adv - adv.mean()) / (adv.std() + 1e-8)
    return obs, act, logp, adv.astype(np.float32), ret


def _worker(rank, world, port, out_path):
    import torch.distributed as dist
    import torch

    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from golden_util import PpoOracle, make_cfg

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    orc = PpoOracle(make_cfg(CFG["obs_dim"], CFG["act_dim"], CFG["hidden"], CFG["num_envs"], num_gpus=2,
                             gmis_per_gpu=1, threads=1))
    orc.rollout()
    g, _ = orc.minibatch(*_minibatch_inputs(orc, rank), gmi=rank)
    t = torch.from_numpy(g.copy())
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    grad_sum = t.numpy()
    orc.adam(grad_sum)
    params = torch.from_numpy(orc.get("params"))
    gathered = [torch.empty_like(params) for _ in range(world)]
    dist.all_gather(gathered, params)
    if rank == 0:
        np.savez(out_path, grad_sum=grad_sum, p0=gathered[0].numpy(), p1=gathered[1].numpy())
    dist.destroy_process_group()


def test_two_rank_gradient_allreduce_matches_single_process(tmp_path):
    import torch.multiprocessing as mp

    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from golden_util import PpoOracle, make_cfg

    out = str(tmp_path / "dist.npz")
    mp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    d = np.load(out)
    # single process: both GMIs of the same job, summed (two terms: order-independent)
    orc = PpoOracle(make_cfg(CFG["obs_dim"], CFG["act_dim"], CFG["hidden"], CFG["num_envs"], num_gpus=2,
                             gmis_per_gpu=1, threads=1))
    orc.rollout()
    g0, _ = orc.minibatch(*_minibatch_inputs(orc, 0), gmi=0)
    g1, _ = orc.minibatch(*_minibatch_inputs(orc, 1), gmi=1)
    assert np.array_equal((g0 + g1).view(np.uint32), d["grad_sum"].view(np.uint32))
    assert np.array_equal(d["p0"].view(np.uint32), d["p1"].view(np.uint32))
    orc.adam(g0 + g1)
    assert np.array_equal(orc.get("params").view(np.uint32), d["p0"].view(np.uint32))


def test_env_partition_is_disjoint_and_complete_across_ranks():
    """GPU-major GMI ids over ranks and [N*c/n, N*(c+1)/n) env slices tile [0, N)."""
    for N, g, t in [(4096, 2, 1), (8192, 8, 4), (32768, 4, 7), (100, 3, 2)]:
        n = g * t
        seen = []
        for rank in range(g):
            for local in range(t):
                c = rank * t + local
                seen.extend(range(N * c // n, N * (c + 1) // n))
        assert seen == list(range(N))


def test_bench_reference_arm_under_torchrun():
    env = dict(os.environ)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.join(ROOT, "bench.py"),
           "--impl", "reference", "--gpus", "2", "--steps", "1", "--warmup", "0", "--envs", "16"]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1  # rank 0 only
    import json
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["value"] > 0 and d["cpu_baseline"]["kind"] == "port"


def test_bench_reference_arm_never_loads_libgmi():
    """The reference arm times the CPU path only: neither the package nor libgmi.so is loaded."""
    code = ("import runpy, sys; sys.argv = ['bench.py', '--impl', 'reference', '--steps', '1', '--warmup', '0', "
            "'--envs', '16']; runpy.run_path('bench.py', run_name='__main__'); "
            "assert 'paper_2206_08482_b200' not in sys.modules; "
            "assert 'libgmi' not in open('/proc/self/maps').read()")
    r = subprocess.run([sys.executable, "-c", code], cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]


def test_async_decoupled_config_validation():
    """decoupled = 2 (AsyncDecoupled across GPUs, mapping.hpp:265-276) is validated before any
    device work: an even num_gpus >= 2 (1:1 serving -> trainer pairs); decoupled in {0, 1, 2}."""
    from paper_2206_08482_b200 import _lib
    from paper_2206_08482_b200.ppo import PpoConfig, Trainer
    base = dict(obs_dim=12, act_dim=3, hidden=[64, 64], num_envs=256)
    for kw, msg in ((dict(num_gpus=1, decoupled=2), "even num_gpus"),
                    (dict(num_gpus=3, rank=1, decoupled=2), "even num_gpus"),
                    (dict(decoupled=3), "decoupled must be")):
        with pytest.raises((_lib.GmiError, ValueError), match=msg):
            Trainer(PpoConfig(**base, **kw))
