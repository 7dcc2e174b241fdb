"""Adaptive GMI manager on hardware: the reference's explore() (Alg. 2,
search.hpp:198-249) driven by measured per-GMI throughput / memory from the B200 PPO
iteration (gmux.GpuProfiler -> gmi_gpu_profile) instead of the synthetic cost model."""
import pytest

pytestmark = pytest.mark.gpu


def test_gpu_profile_point(cuda):
    from paper_2206_08482_b200 import gmux
    p = gmux.GpuProfiler(iters=2)
    r1 = p.profile("AT", 1, 1024)
    assert r1.runnable and r1.top > 0 and r1.mem > 0
    r2 = p.profile("AT", 2, 1024)  # two green-context GMIs, half the SMs each
    assert r2.runnable and r2.top > 0
    # shapes the iteration cannot tile are reported as not runnable, not as errors
    assert not p.profile("AT", 1, 100).runnable
    with pytest.raises(ValueError):
        p.profile("NOPE", 1, 1024)


def test_explore_with_measured_profiles(cuda):
    from paper_2206_08482_b200 import gmux
    w = gmux.load_benchmark("AT")
    est = gmux.ThroughputEstimator(w)
    cfg = gmux.SearchConfig(num_env_grid=[512, 1024, 2048], max_gmis_per_gpu=2)
    res = gmux.explore(gmux.GpuProfiler(iters=2), est, "AT", 1, cfg)
    assert res.feasible and res.gmis_per_gpu in (1, 2) and res.num_env in (512, 1024, 2048)
    assert res.est_throughput > 0
    assert any(v.runnable for v in res.visited)


def test_resize_rebuilds_plans_like_a_fresh_trainer(cuda):
    """gmi_resize on a live trainer (2 green-context GMIs, 32 -> 64 SMs each) gives the same
    GEMM plans as a trainer created at 64 SMs: two iterations agree bit for bit."""
    import numpy as np
    from paper_2206_08482_b200.ppo import PpoConfig, Trainer
    kw = dict(obs_dim=60, act_dim=8, hidden=[256, 256], num_envs=512, gmis_per_gpu=2, gmi_backend=1)
    a = Trainer(PpoConfig(**kw, sm_per_gmi=32))
    a.resize([64, 64])
    b = Trainer(PpoConfig(**kw, sm_per_gmi=64))
    for _ in range(2):
        a.iteration()
        b.iteration()
    assert np.array_equal(a.get("params").view(np.uint32), b.get("params").view(np.uint32))


def test_resize_mid_training_matches_oracle(cuda):
    """Re-splitting between iterations keeps the job's state: after iteration 0 at 16 SMs per
    GMI and iteration 1 at 48, the parameters match the oracle's two iterations."""
    import numpy as np
    from golden_util import PpoOracle, make_cfg
    from paper_2206_08482_b200.ppo import PpoConfig, Trainer
    t = Trainer(PpoConfig(obs_dim=12, act_dim=3, hidden=[64, 64], num_envs=128, gmis_per_gpu=2, gmi_backend=1,
                          sm_per_gmi=16))
    o = PpoOracle(make_cfg(12, 3, [64, 64], 128, gmis_per_gpu=2))
    th0 = o.get("params").astype(np.float64)
    t.iteration()
    o.iteration()
    t.resize([48, 48])
    assert [s for _, s in t.unit_busy()[:2]] == [48, 48]
    t.iteration()
    o.iteration()
    for c in range(2):
        assert np.array_equal(t.get("done", c), o.get("done", c))
    d_dev, d_orc = t.get("params") - th0, o.get("params") - th0
    assert np.linalg.norm(d_dev - d_orc) <= 2e-2 * np.linalg.norm(d_orc)
    with pytest.raises(ValueError):
        t.resize([48, 48, 48])  # the GMI count is fixed (GMI_ERR_INVALID -> ValueError)


def test_tune_serving_share_from_measured_throughput(cuda):
    """Decoupled layout: the manager measures the serving/trainer split candidates on the live
    trainer and keeps the fastest (north_star (3): SM shares retuned from measured throughput)."""
    from paper_2206_08482_b200.ppo import PpoConfig, Trainer
    t = Trainer(PpoConfig(obs_dim=60, act_dim=8, hidden=[256, 256, 256], num_envs=1024, decoupled=1, gmi_backend=1))
    t.iteration()
    cands = [[8, 0], [16, 0], [24, 0]]
    best, tput = t.tune_shares(cands, iters=2)
    assert len(tput) == 3 and all(v > 0 for v in tput)
    assert best == max(range(3), key=lambda i: tput[i])
    assert t.unit_busy()[0][1] == cands[best][0]
    t.iteration()
