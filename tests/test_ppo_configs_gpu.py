"""PPO parity at every BASELINE.json config shape, through libgmi, against the CPU
restatement (oracle/ppo_oracle.c) on the same seeds.

Configs (BASELINE.json `configs`, shapes from workload.hpp:126-134 and SURVEY §8a row a12):
  * configs[0]  AT-like 60:64:64:8, 512 envs, 1 GMI (two iterations: eager, then graph replay)
  * configs[1]  AT-like 60:256:256:256:8, 4096 envs, 1 GMI (the bench workload, full size)
  * configs[2]  HM-like 108:200:400:100:21, 4 green-context GMIs x 1024 envs (rollout, critic,
                GAE, 16 updates with the K1 fold of 4 GMI gradients in the MPR ring order)
  * configs[4]  SH-like 211:512:512:512:256:20 at reduced envs: 2 GMIs x 64 envs and
                7 green-context GMIs x 64 envs (7 x 16 SMs)

Checked per GMI after one iteration (tolerances stated here, asserted below):
  * integer contract, bit-exact: initial parameters, reset masks (done) of every env-step,
    episode counters / clocks (ep_count, ep_step), minibatch permutation indices (the last
    epoch copy's behaviour log-probs equal the rollout's log-probs gathered with the oracle's
    Feistel indices)
  * trajectories over the horizon (T = 32 steps): rewards, observations, actions
    max |d| <= 2e-2 and mean |d| <= 2e-4; advantages / returns max |d| <= 5e-2, mean <= 2e-3
  * loss statistics of the last minibatch of GMI 0 (policy loss, value loss, approx. KL,
    clip fraction): |d| <= 2e-2 * |oracle| + 2e-3 (approx. KL: + 5e-4 absolute)
  * the update: relative parameter-change error ||dtheta_dev - dtheta_orc|| / ||dtheta_orc||
    <= 2e-2 over the whole flat vector and <= 5e-2 per tensor (dtheta = theta_1 - theta_0;
    16 Adam steps at lr 3e-4 move each parameter by at most ~4.8e-3, so raw-theta bounds
    would hide errors of that size)
Residuals: fp32 TMEM accumulation vs the oracle's double sums, SFU ex2/tanh/sin ulps, and the
bf16 rounding flips they cause.
"""
import numpy as np
import pytest

from golden_util import PpoOracle, make_cfg, oracle_perm, param_layout

pytestmark = pytest.mark.gpu

TRAJ = dict(rew=(2e-2, 2e-4), obs=(2e-2, 2e-4), act=(2e-2, 2e-4), adv=(5e-2, 2e-3), ret=(5e-2, 2e-3))


def _make(S, A, hidden, envs, **kw):
    from paper_2206_08482_b200.ppo import PpoConfig, Trainer
    dev = Trainer(PpoConfig(obs_dim=S, act_dim=A, hidden=list(hidden), num_envs=envs, **kw))
    okw = {k: v for k, v in kw.items() if k in ("num_gpus", "gmis_per_gpu", "seed", "horizon", "epochs",
                                                "minibatches")}
    orc = PpoOracle(make_cfg(S, A, hidden, envs, **okw))
    return dev, orc


def _close(name, got, want, max_abs, mean_abs):
    d = np.abs(got.astype(np.float64) - want.astype(np.float64))
    assert d.max() <= max_abs and d.mean() <= mean_abs, (name, float(d.max()), float(d.mean()))
    return float(d.max()), float(d.mean())


def _rel(a, b):
    return float(np.linalg.norm(a - b) / (np.linalg.norm(b) + 1e-30))


def _check_iteration(dev, orc, S, A, hidden, gmis, it, theta0_dev, theta0_orc, s_dev, s_orc):
    report = {}
    for c in range(gmis):
        for f in ("done", "ep_count", "ep_step", "ep_len"):
            assert np.array_equal(dev.get(f, c), orc.get(f, c)), (f, c)
        for f, tol in TRAJ.items():
            report[f"{f}[{c}]"] = _close(f"{f}[{c}]", dev.get(f, c), orc.get(f, c), *tol)
        # permutation indices of the last epoch (Feistel bijection keyed by seed, GMI, iteration, epoch)
        logp = dev.get("trained_logp", c)
        perm = oracle_perm(dev.cfg.seed, dev.cfg.rank * gmis + c, it, dev.cfg.epochs - 1, logp.size)
        assert np.array_equal(dev.get("oldlp_sh", c).view(np.uint32), logp[perm].view(np.uint32)), ("perm", c)
    # loss statistics (last minibatch of GMI 0)
    for f, extra in (("policy_loss", 0.0), ("value_loss", 0.0), ("approx_kl", 5e-4), ("clip_frac", 0.0)):
        a, b = getattr(s_dev, f), getattr(s_orc, f)
        report[f] = (a, b)
        assert abs(a - b) <= 2e-2 * abs(b) + 2e-3 + extra, (f, a, b)
    # relative parameter-change error, whole vector and per tensor
    d_dev = dev.get("params").astype(np.float64) - theta0_dev
    d_orc = orc.get("params").astype(np.float64) - theta0_orc
    report["dtheta"] = _rel(d_dev, d_orc)
    assert report["dtheta"] <= 2e-2, report
    lay = param_layout(S, A, hidden)
    for key, t in lay.items():
        if not isinstance(key, tuple):
            continue
        for part, n in (("w", t["out_p"] * t["in_p"]), ("b", t["out_p"])):
            sl = slice(t[part], t[part] + n)
            if np.linalg.norm(d_orc[sl]) > 0:
                r = _rel(d_dev[sl], d_orc[sl])
                assert r <= 5e-2, (key, part, r)
    ls = slice(lay["log_std"], lay["log_std"] + A)
    assert _rel(d_dev[ls], d_orc[ls]) <= 5e-2
    print(report)
    return report


def _run(S, A, hidden, envs, iters=1, **kw):
    dev, orc = _make(S, A, hidden, envs, **kw)
    gmis = kw.get("gmis_per_gpu", 1)
    assert np.array_equal(dev.get("params").view(np.uint32), orc.get("params").view(np.uint32))
    for it in range(iters):
        t0d, t0o = dev.get("params").astype(np.float64), orc.get("params").astype(np.float64)
        s_dev = dev.iteration()
        s_orc = orc.iteration()
        assert s_dev.env_steps == envs * dev.cfg.horizon
        _check_iteration(dev, orc, S, A, hidden, gmis, it, t0d, t0o, s_dev, s_orc)


def test_config0_at_2x64_512_envs(cuda):
    """BASELINE configs[0]: 60:64:64:8 (P = 16,713), 512 envs, one GMI; iteration 0 eager,
    iteration 1 from the captured CUDA graph."""
    _run(60, 8, [64, 64], 512, iters=2)


def test_config1_at_3x256_4096_envs(cuda):
    """BASELINE configs[1] at full size: 4096 envs, 3x256 (P = 296,713) -- the bench workload's
    kernels (cluster rollout, fused value pass, weight-stationary GEMMs, fused head)."""
    _run(60, 8, [256, 256, 256], 4096, iters=1)


def test_config2_hm_4_green_gmis(cuda):
    """BASELINE configs[2] layout: HM 108:200:400:100:21 (P = 286,822), 4 GMIs on SM-partitioned
    green contexts (gmi_backend = 1) with 1024 envs each; the update folds the 4 GMI gradients
    with K1 before every Adam step."""
    _run(108, 21, [200, 400, 100], 4096, iters=1, gmis_per_gpu=4, gmi_backend=1)


@pytest.mark.parametrize("gmis,backend", [(2, 0), (7, 1)])
def test_config4_sh_gmis(cuda, gmis, backend):
    """BASELINE configs[4] shapes: SH 211:512:512:512:256:20 (P = 1,535,765) at 64 envs per GMI,
    2 GMIs (streams) and 7 GMIs (7 x 16-SM green contexts)."""
    _run(211, 20, [512, 512, 512, 256], 64 * gmis, iters=1, gmis_per_gpu=gmis, gmi_backend=backend)


def test_config4_sh_wide_weight_stationary(cuda):
    """SH widths at 1024 envs on one GMI: enough minibatch rows for every CTA to get a tile, so
    the 512-wide input gradient with K = 256 (dPre_3 -> dH_2) takes the wide weight-stationary
    GEMM (128-column parts of dPre_2, the part's weights resident)."""
    _run(211, 20, [512, 512, 512, 256], 1024, iters=1)


@pytest.mark.parametrize("serving_sms", [16, 32])
def test_decoupled_wide_nets_match_oracle(cuda, serving_sms):
    """Decoupled layout with HM-width nets (108:200:400:100:21): the serving GMI runs the
    per-layer rollout / value path on its partition (the fused kernels hold <= 256 widths) with
    the policy snapshot; two iterations against the oracle's lagged schedule."""
    S, A, hidden = 108, 21, [200, 400, 100]
    dev, orc = _make(S, A, hidden, 256, decoupled=1, gmi_backend=1, serving_sms=serving_sms)
    th0 = orc.get("params").astype(np.float64)
    for it in range(2):
        dev.iteration()
        orc.iteration_decoupled()
        assert np.array_equal(dev.get("done"), orc.get("done")), it
        for f in ("rew", "adv"):
            _close(f"{f}[{it}]", dev.get(f), orc.get(f), *TRAJ[f])
    d_dev = dev.get("params").astype(np.float64) - th0
    d_orc = orc.get("params").astype(np.float64) - th0
    assert _rel(d_dev, d_orc) <= 2e-2, _rel(d_dev, d_orc)
