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
