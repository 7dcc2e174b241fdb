"""Multi-rank data-parallel PPO through libgmi on one B200: several ranks of one job wired with
the peer exchange (cfg.comm = 1, cuda/exchange.cu: fused reduce-scatter -> sharded Adam ->
all-gather over peer memory, the HAR leader step of reduction.hpp:287-299).

Every gpurun box has one GPU, so the ranks live in one process on cuda:0 and are wired with
gmi_ppo_comm_connect (the same kernels, flags and fold order as one process per GPU over
CUDA IPC; only the pointer source differs). Checks:
  * 2 ranks x 1 GMI == 1 rank x 2 GMIs, bit for bit (same env slices, RNG keys, permutation
    keys; the leader-ring fold of 2 ranks is the MPR fold of 2 GMIs; same Adam arithmetic), and
    both ranks hold bit-identical parameters;
  * 2 ranks x 2 GMIs against the oracle's 2-GPU layout (leader-ring fold over per-GPU rings):
    integer state bit-exact, relative parameter-change error <= 2e-2;
  * the exchange over a single rank is bit-identical to the plain Adam kernel (3 iterations:
    eager, then CUDA-graph replays), for 1 GMI, 2 GMIs and the decoupled layout;
  * an unwired rank (decomposition hooks only): its env slice, reset masks and rollout equal
    the oracle's GMI of that rank, and gmi_ppo_iteration refuses to run.
"""
import numpy as np
import pytest

from golden_util import PpoOracle, make_cfg

pytestmark = [pytest.mark.gpu, pytest.mark.timeout(300)]

SMALL = dict(obs_dim=12, act_dim=3, hidden=[64, 64])


def _ranks(n, envs, gmis=1, **kw):
    from paper_2206_08482_b200.ppo import PpoConfig, Trainer
    ts = [Trainer(PpoConfig(**SMALL, num_envs=envs, num_gpus=n, rank=r, gmis_per_gpu=gmis, comm=1, **kw))
          for r in range(n)]
    Trainer.comm_connect(ts)
    return ts


def _iterate(ts, iters):
    for _ in range(iters):
        for t in ts:
            t.iteration_async()
        stats = [t.synchronize() for t in ts]
    return stats


def test_two_ranks_equal_one_rank_two_gmis(cuda):
    from paper_2206_08482_b200.ppo import PpoConfig, Trainer
    ranks = _ranks(2, 128)
    one = Trainer(PpoConfig(**SMALL, num_envs=128, gmis_per_gpu=2))
    _iterate(ranks, 3)
    for _ in range(3):
        one.iteration()
    p0, p1, p = (x.get("params").view(np.uint32) for x in (ranks[0], ranks[1], one))
    assert np.array_equal(p0, p1)
    assert np.array_equal(p0, p)
    for r in range(2):
        for f in ("done", "ep_count", "rew", "act"):
            assert np.array_equal(ranks[r].get(f), one.get(f, r)), (r, f)


def test_two_ranks_two_gmis_match_oracle(cuda):
    ranks = _ranks(2, 256, gmis=2)
    orc = PpoOracle(make_cfg(12, 3, [64, 64], 256, num_gpus=2, gmis_per_gpu=2))
    th0 = orc.get("params").astype(np.float64)
    assert np.array_equal(ranks[0].get("params").view(np.uint32), orc.get("params").view(np.uint32))
    _iterate(ranks, 1)
    orc.iteration()
    for r in range(2):
        for c in range(2):
            for f in ("done", "ep_count", "ep_step"):
                assert np.array_equal(ranks[r].get(f, c), orc.get(f, 2 * r + c)), (r, c, f)
    assert np.array_equal(ranks[0].get("params").view(np.uint32), ranks[1].get("params").view(np.uint32))
    d_dev = ranks[0].get("params").astype(np.float64) - th0
    d_orc = orc.get("params").astype(np.float64) - th0
    rel = np.linalg.norm(d_dev - d_orc) / np.linalg.norm(d_orc)
    assert rel <= 2e-2, rel


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
        with pytest.raises(_lib.GmiError):
            t.iteration()
