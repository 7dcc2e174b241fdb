"""Multi-rank data-parallel PPO through libgmi on one B200: several ranks of one job wired with
the peer exchange (cfg.comm = 1, cuda/exchange.cu: fused reduce-scatter -> sharded Adam ->
all-gather over peer memory, the HAR leader step of reduction.hpp:287-299).

Every gpurun box has one GPU, so the ranks are separate processes on cuda:0 (one CUDA context
each, time-sliced) wired over CUDA IPC exactly as one process per GPU would be
(tests/multirank_worker.py: gmi_ppo_comm_handle -> gloo all_gather_object ->
gmi_ppo_comm_attach). Checks:
  * 2 ranks x 1 GMI == 1 rank x 2 GMIs, bit for bit (same env slices, RNG keys, permutation
    keys; the leader-ring fold of 2 ranks is the MPR fold of 2 GMIs; same Adam arithmetic), and
    both ranks hold bit-identical parameters;
  * 2 ranks x 2 GMIs (MRR) and 3 ranks x 4 GMIs (HAR) against the oracle's layouts:
    integer state bit-exact, relative parameter-change error <= 2e-2;
  * the exchange over a single rank is bit-identical to the plain Adam kernel (3 iterations:
    eager, then CUDA-graph replays), for 1 GMI, 2 GMIs and the decoupled layout;
  * an unwired rank (decomposition hooks only): its env slice, reset masks and rollout equal
    the oracle's GMI of that rank, and gmi_ppo_iteration refuses to run.
"""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

from golden_util import PpoOracle, make_cfg

pytestmark = [pytest.mark.gpu, pytest.mark.timeout(600)]

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SMALL = dict(obs_dim=12, act_dim=3, hidden=[64, 64])


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _job(tmp_path, world, envs, gmis=1, iters=2, decoupled=0, split=0, backend=-1):
    """Runs `world` rank processes on cuda:0 and returns their dumps."""
    port = _port()
    procs, outs = [], []
    for r in range(world):
        out = str(tmp_path / f"rank{r}.npz")
        outs.append(out)
        procs.append(subprocess.Popen([sys.executable, os.path.join(ROOT, "tests", "multirank_worker.py"),
                                       "--rank", str(r), "--world", str(world), "--port", str(port),
                                       "--envs", str(envs), "--gmis", str(gmis), "--iters", str(iters),
                                       "--decoupled", str(decoupled), "--split", str(split),
                                       "--backend", str(backend),
                                       "--out", out], cwd=ROOT, stdout=subprocess.PIPE, stderr=subprocess.STDOUT,
                                      text=True))
    logs = []
    try:
        for p in procs:
            logs.append(p.communicate(timeout=400)[0])
    finally:
        for p in procs:
            if p.poll() is None:
                p.kill()
    for p, log in zip(procs, logs):
        assert p.returncode == 0, log[-3000:]
    return [dict(np.load(o)) for o in outs]


def test_two_ranks_equal_one_rank_two_gmis(cuda, tmp_path):
    from paper_2206_08482_b200.ppo import PpoConfig, Trainer
    ranks = _job(tmp_path, 2, 128, iters=2)
    one = Trainer(PpoConfig(**SMALL, num_envs=128, gmis_per_gpu=2))
    for _ in range(2):
        one.iteration()
    p = one.get("params").view(np.uint32)
    assert np.array_equal(ranks[0]["params"].view(np.uint32), ranks[1]["params"].view(np.uint32))
    assert np.array_equal(ranks[0]["params"].view(np.uint32), p)
    for r in range(2):
        for f in ("done", "ep_count", "rew", "act"):
            assert np.array_equal(ranks[r][f"{f}0"], one.get(f, r)), (r, f)


def test_two_ranks_two_gmis_match_oracle(cuda, tmp_path):
    """2 GPUs x 2 GMIs: Alg. 1 selects MRR (t <= g), so the exchange folds two rings of one GMI
    per rank; the oracle folds the same way."""
    ranks = _job(tmp_path, 2, 256, gmis=2, iters=1)
    orc = PpoOracle(make_cfg(12, 3, [64, 64], 256, num_gpus=2, gmis_per_gpu=2))
    th0 = orc.get("params").astype(np.float64)
    orc.iteration()
    for r in range(2):
        for c in range(2):
            for f in ("done", "ep_count", "ep_step"):
                assert np.array_equal(ranks[r][f"{f}{c}"], orc.get(f, 2 * r + c)), (r, c, f)
    assert np.array_equal(ranks[0]["params"].view(np.uint32), ranks[1]["params"].view(np.uint32))
    d_dev = ranks[0]["params"].astype(np.float64) - th0
    d_orc = orc.get("params").astype(np.float64) - th0
    rel = np.linalg.norm(d_dev - d_orc) / np.linalg.norm(d_orc)
    assert rel <= 2e-2, rel


def test_three_ranks_har_match_oracle(cuda, tmp_path):
    """3 GPUs x 4 GMIs: t > g, so Alg. 1 selects HAR -- K1 folds per rank, then the leaders'
    ring over the three ranks."""
    ranks = _job(tmp_path, 3, 3 * 4 * 16, gmis=4, iters=1)
    orc = PpoOracle(make_cfg(12, 3, [64, 64], 3 * 4 * 16, num_gpus=3, gmis_per_gpu=4))
    th0 = orc.get("params").astype(np.float64)
    orc.iteration()
    for r in range(3):
        assert np.array_equal(ranks[r]["params"].view(np.uint32), ranks[0]["params"].view(np.uint32))
        for c in range(4):
            assert np.array_equal(ranks[r][f"done{c}"], orc.get("done", 4 * r + c)), (r, c)
    d_dev = ranks[0]["params"].astype(np.float64) - th0
    d_orc = orc.get("params").astype(np.float64) - th0
    assert np.linalg.norm(d_dev - d_orc) <= 2e-2 * np.linalg.norm(d_orc)


def test_two_ranks_decoupled_match_oracle(cuda, tmp_path):
    """BASELINE configs[3] shape on 2 GPUs: per GPU a serving GMI (16-SM green context) streams
    experience to the trainer GMI; the trainer GMIs' gradients cross GPUs through the peer
    exchange. Two iterations against the oracle's lagged schedule with num_gpus = 2."""
    ranks = _job(tmp_path, 2, 128, iters=2, decoupled=1)
    orc = PpoOracle(make_cfg(12, 3, [64, 64], 128, num_gpus=2))
    th0 = orc.get("params").astype(np.float64)
    for _ in range(2):
        orc.iteration_decoupled()
    assert np.array_equal(ranks[0]["params"].view(np.uint32), ranks[1]["params"].view(np.uint32))
    for r in range(2):
        assert np.array_equal(ranks[r]["done0"], orc.get("done", r)), r
    d_dev = ranks[0]["params"].astype(np.float64) - th0
    d_orc = orc.get("params").astype(np.float64) - th0
    assert np.linalg.norm(d_dev - d_orc) <= 2e-2 * np.linalg.norm(d_orc)


@pytest.mark.parametrize("layout", [dict(gmis_per_gpu=1), dict(gmis_per_gpu=2), dict(decoupled=1, gmi_backend=1)])
def test_single_rank_exchange_equals_adam_kernel(cuda, layout):
    from paper_2206_08482_b200.ppo import PpoConfig, Trainer
    a = Trainer(PpoConfig(**SMALL, num_envs=64, **layout))
    b = Trainer(PpoConfig(**SMALL, num_envs=64, comm=1, **layout))
    for _ in range(3):
        a.iteration()
        b.iteration()
    assert np.array_equal(a.get("params").view(np.uint32), b.get("params").view(np.uint32))


def test_unwired_rank_hooks_match_oracle_slice(cuda):
    from paper_2206_08482_b200 import _lib
    from paper_2206_08482_b200.ppo import PpoConfig, Trainer
    orc = PpoOracle(make_cfg(12, 3, [64, 64], 128, num_gpus=2))
    ts = [Trainer(PpoConfig(**SMALL, num_envs=128, num_gpus=2, rank=r, comm=1)) for r in range(2)]
    for r, t in enumerate(ts):  # env slice [N r/2, N (r+1)/2): initial state and episode clocks
        for f in ("x", "ep_len", "ep_step"):
            assert np.array_equal(t.get(f), orc.get(f, r)), (r, f)
    orc.rollout()
    for r, t in enumerate(ts):
        t.rollout()
        for f in ("done", "ep_count", "ep_step"):
            assert np.array_equal(t.get(f), orc.get(f, r)), (r, f)
        d = np.abs(t.get("rew").astype(np.float64) - orc.get("rew", r))
        assert d.max() <= 2e-2 and d.mean() <= 2e-4
        with pytest.raises((_lib.GmiError, ValueError)):
            t.iteration()
    with pytest.raises((_lib.GmiError, ValueError)):  # ranks sharing a device need a process each
        Trainer.comm_connect(ts)


def test_bench_two_ranks_on_one_gpu(cuda):
    """The driver's N > 1 bench path (torchrun, one rank per GPU, peer exchange wired over CUDA
    IPC, max-over-ranks timing, one JSON line) run as 2 rank processes sharing cuda:0
    (GMI_BENCH_SHARE_GPU=1: time-sliced, so the number is not a measurement)."""
    import json
    env = dict(os.environ, GMI_BENCH_SHARE_GPU="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", str(_port()), os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "2",
           "--warmup", "3", "--envs", "256", "--no-cpu-baseline", "--no-multi-gmi"]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=500)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["run"]["comm"].startswith("peer exchange")
    assert d["config"]["envs_per_gpu"] == 256


def test_bench_async_decoupled_two_ranks_on_one_gpu(cuda):
    """bench.py --decoupled 2 --gpus 2: serving rank 0 and trainer rank 1 wired over the link
    windows, env-steps summed over ranks (serving only), rank 0 reports the trainer's phases
    (GMI_BENCH_SHARE_GPU=1: both ranks on cuda:0, time-sliced, not a measurement)."""
    import json
    env = dict(os.environ, GMI_BENCH_SHARE_GPU="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", str(_port()), os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "2",
           "--warmup", "3", "--envs", "256", "--decoupled", "2", "--no-cpu-baseline", "--no-multi-gmi"]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=500)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["run"]["decoupled_mode"].startswith("across GPUs")
    assert d["run"]["env_steps_per_step"] == 256 * 32
    assert d["phases"]["fwd_gemm"]["launches"] > 0  # the trainer rank's profile


@pytest.mark.parametrize("world", [2, 4])
def test_async_decoupled_across_ranks(cuda, tmp_path, world):
    """AsyncDecoupled across GPUs (decoupled = 2, mapping.hpp:265-276): serving rank s rolls out
    env slice s of G/2 on a whole GPU; trainer rank G/2 + s pulls each rollout from the partner's
    link window, trains (the trainer ranks form a G/2-rank data-parallel job over the peer
    exchange) and pushes the policy snapshot back -- device flags, one-iteration policy lag.
    Must equal the colocated decoupled job with G/2 GPUs (decoupled = 1, whole-GPU streams) bit
    for bit: trainer parameters, every serving rank's snapshot (theta_K after the last push) and
    latest rollout; env-steps are counted by the serving ranks only."""
    iters, envs, half = 3, 256, world // 2
    ranks = _job(tmp_path, world, envs, iters=iters, split=1)
    if half == 1:
        from paper_2206_08482_b200.ppo import PpoConfig, Trainer
        one = Trainer(PpoConfig(**SMALL, num_envs=envs, decoupled=1, gmi_backend=0))
        for _ in range(iters):
            one.iteration()
        ref = [{"params": one.get("params"), **{f"{f}0": one.get(f) for f in ("done", "rew", "act")}}]
    else:
        (tmp_path / "ref").mkdir()
        ref = _job(tmp_path / "ref", half, envs, iters=iters, decoupled=1, backend=0)
    for s in range(half):
        sv, tr = ranks[s], ranks[half + s]
        p = ref[s]["params"].view(np.uint32)
        assert np.array_equal(tr["params"].view(np.uint32), p), s
        assert np.array_equal(sv["params"].view(np.uint32), p), s  # snapshot pushed by the trainer
        for f in ("done", "rew", "act"):
            assert np.array_equal(sv[f], ref[s][f"{f}0"]), (s, f)  # latest rollout (K + 1 on both)
        assert list(sv["steps"]) == [envs // half * 32] * iters and list(tr["steps"]) == [0] * iters
