"""B200 PPO iteration (libgmi) vs the CPU restatement (oracle/ppo_oracle.c).

Tolerances (stated per quantity; the oracle mirrors every bf16 rounding point, so the
residual is fp32 accumulation order in TMEM vs double on the CPU, ulp differences of
expf/logf/tanhf/sinf, and the occasional bf16 rounding flip those cause):
  * integer state (episode clocks, reset masks) and initial parameters: bit-exact
  * rollout trajectories over the horizon: max |d| <= 2e-2, mean |d| <= 1e-4 (act/obs/rew)
  * minibatch gradients: per tensor ||d|| <= 2e-2 ||g||
  * parameters after one full iteration (16 Adam steps, lr 3e-4): max |d| <= 2e-3, mean |d| <= 5e-5
"""
import numpy as np
import pytest

from golden_util import PpoOracle, make_cfg, param_layout

pytestmark = pytest.mark.gpu

SMALL = dict(obs_dim=12, act_dim=3, hidden=[64, 64], num_envs=64)


def _pair(obs_dim, act_dim, hidden, num_envs, **kw):
    from paper_2206_08482_b200.ppo import PpoConfig, Trainer
    dev = Trainer(PpoConfig(obs_dim=obs_dim, act_dim=act_dim, hidden=list(hidden), num_envs=num_envs, **kw))
    okw = {k: v for k, v in kw.items() if k in ("num_gpus", "gmis_per_gpu", "seed", "horizon", "epochs",
                                                "minibatches", "lr", "ent_coef", "vf_coef")}
    orc = PpoOracle(make_cfg(obs_dim, act_dim, hidden, num_envs, **okw))
    return dev, orc


def _close(name, got, want, max_abs, mean_abs):
    d = np.abs(got.astype(np.float64) - want.astype(np.float64))
    assert d.max() <= max_abs and d.mean() <= mean_abs, (name, float(d.max()), float(d.mean()))


def test_init_is_bit_exact(cuda):
    dev, orc = _pair(**SMALL)
    assert dev.param_count == orc.P
    assert np.array_equal(dev.get("params").view(np.uint32), orc.get("params").view(np.uint32))
    for f in ("x", "ep_len", "ep_step"):
        assert np.array_equal(dev.get(f), orc.get(f)), f


@pytest.mark.parametrize("gmis", [1, 2])
def test_rollout_matches_oracle(cuda, gmis):
    dev, orc = _pair(**SMALL, gmis_per_gpu=gmis)
    dev.rollout()
    orc.rollout()
    for c in range(gmis):
        assert np.array_equal(dev.get("done", c), orc.get("done", c))
        assert np.array_equal(dev.get("ep_count", c), orc.get("ep_count", c))
        _close("act", dev.get("act", c), orc.get("act", c), 2e-2, 1e-4)
        _close("obs", dev.get("obs", c), orc.get("obs", c), 2e-2, 1e-4)
        _close("rew", dev.get("rew", c), orc.get("rew", c), 2e-2, 1e-4)
        _close("logp", dev.get("logp", c), orc.get("logp", c), 5e-2, 1e-3)
        _close("val", dev.get("val", c), orc.get("val", c), 2e-2, 1e-4)
        _close("adv", dev.get("adv", c), orc.get("adv", c), 5e-2, 1e-3)
        _close("ret", dev.get("ret", c), orc.get("ret", c), 5e-2, 1e-3)


@pytest.mark.parametrize("dims", [(12, 3, [64, 64]), (60, 8, [256, 256, 256]), (108, 21, [200, 400, 100])])
def test_minibatch_gradient_matches_oracle(cuda, dims):
    S, A, hidden = dims
    dev, orc = _pair(S, A, hidden, 64)
    B = 64 * 32 // 4
    rng = np.random.default_rng(S)
    X = rng.uniform(-1, 1, (B, S)).astype(np.float32)
    act = rng.standard_normal((B, A)).astype(np.float32)
    oldlp = (rng.standard_normal(B) - 3).astype(np.float32)
    adv = rng.standard_normal(B).astype(np.float32)
    ret = rng.standard_normal(B).astype(np.float32)
    g_dev = dev.minibatch_grad(X, act, oldlp, adv, ret)
    g_orc, _ = orc.minibatch(X, act, oldlp, adv, ret)
    lay = param_layout(S, A, hidden)
    for key, t in lay.items():
        if not isinstance(key, tuple):
            continue
        for part, n in (("w", t["out_p"] * t["in_p"]), ("b", t["out_p"])):
            a, b = g_dev[t[part]:t[part] + n], g_orc[t[part]:t[part] + n]
            ref = np.linalg.norm(b) + 1e-12
            assert np.linalg.norm(a - b) <= 2e-2 * ref, (key, part, np.linalg.norm(a - b) / ref)
    ls = slice(lay["log_std"], lay["log_std"] + A)
    assert np.linalg.norm(g_dev[ls] - g_orc[ls]) <= 2e-2 * (np.linalg.norm(g_orc[ls]) + 1e-12)


@pytest.mark.parametrize("gmis", [1, 2])
def test_full_iteration_matches_oracle(cuda, gmis):
    dev, orc = _pair(**SMALL, gmis_per_gpu=gmis)
    s = dev.iteration()
    orc.iteration()
    assert s.env_steps == SMALL["num_envs"] * 32
    _close("params", dev.get("params"), orc.get("params"), 2e-3, 5e-5)
    m_dev, m_orc = dev.get("adam_m"), orc.get("adam_m")
    assert np.linalg.norm(m_dev - m_orc) <= 5e-2 * np.linalg.norm(m_orc)
    # the next rollout starts from the carried-over observation slot
    dev.rollout()
    orc.rollout()
    assert np.array_equal(dev.get("done"), orc.get("done"))
    _close("rew", dev.get("rew"), orc.get("rew"), 5e-2, 5e-4)


def test_iterations_are_deterministic(cuda):
    from paper_2206_08482_b200.ppo import PpoConfig, Trainer
    runs = []
    for _ in range(2):
        t = Trainer(PpoConfig(obs_dim=12, act_dim=3, hidden=[64, 64], num_envs=64, gmis_per_gpu=2))
        t.iteration()
        t.iteration()
        runs.append(t.get("params"))
    assert np.array_equal(runs[0].view(np.uint32), runs[1].view(np.uint32))


@pytest.mark.parametrize("chain", ["1", "0"])
def test_repeated_runs_are_bit_identical_at_bench_shape(cuda, monkeypatch, chain):
    """Eight fresh trainers at the bench shape (AT 3x256, 4096 envs), two iterations each, end
    bit-identical. Regression for a lapping race in the fused head kernel (a loss warp running a
    tile ahead completed the count-4 G-ready barrier while a slower warp's G rows were unwritten):
    ~1 run in 6 differed (tools/determinism_stress.py, profiles/r2/SUMMARY.md)."""
    from paper_2206_08482_b200.ppo import PpoConfig, Trainer
    monkeypatch.setenv("GMI_FWD_CHAIN", chain)
    ref = None
    for _ in range(8):
        t = Trainer(PpoConfig(obs_dim=60, act_dim=8, hidden=[256, 256, 256], num_envs=4096))
        t.iteration()
        t.iteration()
        p = t.get("params").view(np.uint32).copy()
        del t
        if ref is None:
            ref = p
        assert np.array_equal(p, ref)


def test_rollout_is_layout_invariant_on_device(cuda):
    from paper_2206_08482_b200.ppo import PpoConfig, Trainer
    one = Trainer(PpoConfig(obs_dim=12, act_dim=3, hidden=[64, 64], num_envs=64))
    two = Trainer(PpoConfig(obs_dim=12, act_dim=3, hidden=[64, 64], num_envs=64, gmis_per_gpu=2))
    one.rollout()
    two.rollout()
    r1 = one.get("rew").reshape(32, 64)
    r2 = np.concatenate([two.get("rew", c).reshape(32, 32) for c in range(2)], axis=1)
    assert np.array_equal(r1, r2)


@pytest.mark.parametrize("env", [None, "GMI_DW_GROUP=0", "GMI_DX_WS4_OFF=1"])
def test_minibatch_gradient_bench_kernels_match_oracle(cuda, monkeypatch, env):
    """Minibatch large enough (1200 envs: 9600 rows, 75 M-tiles per net) that the plan picks the
    bench's kernels: weight-stationary forward GEMMs, the 4-problem weight-stationary input
    gradient (N-halves), and the grouped weight gradient of layers 2+1 (18 splits); the
    non-default plans stay covered through their switches."""
    if env:
        k, v = env.split("=")
        monkeypatch.setenv(k, v)
    S, A, hidden = 60, 8, [256, 256, 256]
    dev, orc = _pair(S, A, hidden, 1200)
    B = 1200 * 32 // 4
    rng = np.random.default_rng(7)
    X = rng.uniform(-1, 1, (B, S)).astype(np.float32)
    act = rng.standard_normal((B, A)).astype(np.float32)
    oldlp = (rng.standard_normal(B) - 3).astype(np.float32)
    adv = rng.standard_normal(B).astype(np.float32)
    ret = rng.standard_normal(B).astype(np.float32)
    g_dev = dev.minibatch_grad(X, act, oldlp, adv, ret)
    g_orc, _ = orc.minibatch(X, act, oldlp, adv, ret)
    lay = param_layout(S, A, hidden)
    for key, t in lay.items():
        if not isinstance(key, tuple):
            continue
        for part, n in (("w", t["out_p"] * t["in_p"]), ("b", t["out_p"])):
            a, b = g_dev[t[part]:t[part] + n], g_orc[t[part]:t[part] + n]
            ref = np.linalg.norm(b) + 1e-12
            assert np.linalg.norm(a - b) <= 2e-2 * ref, (key, part, np.linalg.norm(a - b) / ref)


@pytest.mark.parametrize("dims", [(12, 3, [64, 64]), (60, 8, [256, 256, 256]), (40, 20, [96, 160]),
                                  (108, 21, [200, 400, 100]), (40, 20, [96, 448, 160, 64])])
def test_fused_rollout_matches_per_layer_path(cuda, monkeypatch, dims):
    """cuda/rollout.cu (one persistent kernel) vs the per-layer GEMM + act/env path: the MLP
    arithmetic is identical, so integer state, actions and observations agree bit-for-bit;
    rewards / log-probs differ only in the order of their small reductions. The last two shapes
    (HM 108:200:400:100 and a 4-layer net) take the wide variant (rollout_kernel<8, true>,
    value_mlp_kernel<true>: 128-row weight parts, TMEM accumulators that wait for the previous
    layer's drain where they overlap)."""
    from paper_2206_08482_b200.ppo import PpoConfig, Trainer
    S, A, hidden = dims
    cfg = dict(obs_dim=S, act_dim=A, hidden=hidden, num_envs=200)
    fused = Trainer(PpoConfig(**cfg))
    monkeypatch.setenv("GMI_ROLLOUT_UNFUSED", "1")
    monkeypatch.setenv("GMI_VALUE_UNFUSED", "1")
    plain = Trainer(PpoConfig(**cfg))
    for it in range(2):  # second rollout starts from the carried-over observation slot
        if it:  # train on the hook's rollout, then give both the same weights
            fused.iteration()
            plain.iteration()
            plain.set("params", fused.get("params"))
        fused.rollout()
        plain.rollout()
        for f in ("done", "ep_count", "ep_step", "act", "obs", "x", "val"):
            assert np.array_equal(fused.get(f), plain.get(f)), f
        for f in ("rew", "logp"):
            np.testing.assert_allclose(fused.get(f), plain.get(f), rtol=1e-5, atol=1e-5)
    # the fused path really ran: one rollout + one value launch instead of T x (L + 2) + ...
    assert fused.synchronize().kernel_launches < plain.synchronize().kernel_launches


def _grad_pair(monkeypatch, env_first, env_second, dims, envs=200):
    from paper_2206_08482_b200.ppo import PpoConfig, Trainer
    S, A, hidden = dims
    cfg = dict(obs_dim=S, act_dim=A, hidden=hidden, num_envs=envs)
    if env_first:
        monkeypatch.setenv(env_first, "1")
    fused = Trainer(PpoConfig(**cfg))
    if env_first:
        monkeypatch.delenv(env_first)
    if env_second:
        monkeypatch.setenv(env_second, "1")
    plain = Trainer(PpoConfig(**cfg))
    B = envs * 32 // 4
    rng = np.random.default_rng(S + A)
    X = rng.uniform(-1, 1, (B, S)).astype(np.float32)
    act = rng.standard_normal((B, A)).astype(np.float32)
    oldlp = (rng.standard_normal(B) - 3).astype(np.float32)
    adv = rng.standard_normal(B).astype(np.float32)
    ret = rng.standard_normal(B).astype(np.float32)
    return fused.minibatch_grad(X, act, oldlp, adv, ret), plain.minibatch_grad(X, act, oldlp, adv, ret)


@pytest.mark.parametrize("dims", [(60, 8, [256, 256, 256]), (12, 3, [64]), (40, 20, [96, 160, 64]),
                                  (100, 1, [128, 256, 192])])
def test_fused_train_forward_matches_per_layer_path(cuda, monkeypatch, dims):
    """cuda/train_fwd.cu (all hidden layers on chip + the fused head step, one launch per
    minibatch) vs per-layer forward GEMMs + the fused head kernel. Same operands, MMA K order,
    bias/ELU and loss code; only the head weight-gradient summation order (per-tile fp32
    partials in registers vs one TMEM accumulator) differs. 1000 rows: a ragged last tile."""
    S, A, hidden = dims
    g1, g2 = _grad_pair(monkeypatch, "GMI_TRAIN_FWD", None, dims, envs=1000)
    lay = param_layout(S, A, hidden)
    for key, t in lay.items():
        if not isinstance(key, tuple):
            continue
        for part, n in (("w", t["out_p"] * t["in_p"]), ("b", t["out_p"])):
            a, b = g1[t[part]:t[part] + n], g2[t[part]:t[part] + n]
            assert np.linalg.norm(a - b) <= 1e-5 * (np.linalg.norm(b) + 1e-12), (key, part)
    ls = slice(lay["log_std"], lay["log_std"] + A)
    np.testing.assert_allclose(g1[ls], g2[ls], rtol=1e-5, atol=1e-7)


@pytest.mark.parametrize("dims", [(12, 3, [64, 64]), (60, 8, [256, 256, 256]), (40, 20, [96, 160])])
def test_fused_head_matches_per_kernel_path(cuda, monkeypatch, dims):
    """cuda/head_fused.cu (head forward + loss + head input / weight gradients + bias sums in
    one kernel) vs the head GEMMs + loss kernel path on the same minibatch. The per-row loss
    and every bf16 rounding point are shared; only fp32 accumulation orders differ."""
    from paper_2206_08482_b200.ppo import PpoConfig, Trainer
    S, A, hidden = dims
    cfg = dict(obs_dim=S, act_dim=A, hidden=hidden, num_envs=200)
    fused = Trainer(PpoConfig(**cfg))
    monkeypatch.setenv("GMI_HEAD_UNFUSED", "1")
    plain = Trainer(PpoConfig(**cfg))
    B = 200 * 32 // 4
    rng = np.random.default_rng(S + A)
    X = rng.uniform(-1, 1, (B, S)).astype(np.float32)
    act = rng.standard_normal((B, A)).astype(np.float32)
    oldlp = (rng.standard_normal(B) - 3).astype(np.float32)
    adv = rng.standard_normal(B).astype(np.float32)
    ret = rng.standard_normal(B).astype(np.float32)
    g1 = fused.minibatch_grad(X, act, oldlp, adv, ret)
    g2 = plain.minibatch_grad(X, act, oldlp, adv, ret)
    lay = param_layout(S, A, hidden)
    for key, t in lay.items():
        if not isinstance(key, tuple):
            continue
        for part, n in (("w", t["out_p"] * t["in_p"]), ("b", t["out_p"])):
            a, b = g1[t[part]:t[part] + n], g2[t[part]:t[part] + n]
            assert np.linalg.norm(a - b) <= 1e-4 * (np.linalg.norm(b) + 1e-12), (key, part)
    ls = slice(lay["log_std"], lay["log_std"] + A)
    np.testing.assert_allclose(g1[ls], g2[ls], rtol=1e-4, atol=1e-7)


def test_bench_workload_runs(cuda):
    """BASELINE config 2: AT, 4096 envs, 3x256, 1 GMI."""
    from paper_2206_08482_b200.ppo import PpoConfig, Trainer
    t = Trainer(PpoConfig.from_benchmark("AT", 4096, hidden=[256, 256, 256], instrument=1))
    assert t.real_param_count == 296713
    for _ in range(2):
        s = t.iteration()
    assert s.env_steps == 4096 * 32
    assert np.isfinite([s.policy_loss, s.value_loss, s.approx_kl, s.mean_reward]).all()
    assert s.gemm_launches > 0 and s.kernel_launches > s.gemm_launches
    assert np.isfinite(t.get("params")).all()


@pytest.mark.parametrize("backend", [0, 1])
def test_decoupled_mode_matches_oracle(cuda, backend):
    """Decoupled mode (BASELINE config 4 on one GPU): a serving GMI (16-SM green context, or a
    plain stream) rolls out, evaluates the critic and runs GAE into the experience channel with
    the policy snapshot while the trainer GMI trains on the previous rollout. Three iterations (the first eager, then CUDA
    graph replays) against the oracle's lagged schedule; same tolerances as the synchronous
    iteration, reset masks bit-exact."""
    dev, orc = _pair(**SMALL, decoupled=1, gmi_backend=backend)
    for it in range(3):
        s = dev.iteration()
        o = orc.iteration_decoupled()
        assert s.env_steps == SMALL["num_envs"] * 32
        tol = (2e-3, 5e-5) if it == 0 else (4e-3, 1e-4)
        _close(f"params[{it}]", dev.get("params"), orc.get("params"), *tol)
        # reset masks of the latest rollout (the channel, one ahead of the trainer): bit-exact
        assert np.array_equal(dev.get("done"), orc.get("done")), it
        _close(f"rew[{it}]", dev.get("rew"), orc.get("rew"), 5e-2, 5e-4)
        _close(f"adv[{it}]", dev.get("adv"), orc.get("adv"), 5e-2, 5e-4)  # serving-side critic + GAE
        assert abs(s.mean_reward - o.mean_reward) < 1e-3


def test_decoupled_bench_shape_matches_oracle(cuda):
    dev, orc = _pair(60, 8, [256, 256, 256], 128, decoupled=1, gmi_backend=1)
    for it in range(2):
        dev.iteration()
        orc.iteration_decoupled()
        _close(f"params[{it}]", dev.get("params"), orc.get("params"), 4e-3, 1e-4)


@pytest.mark.parametrize("layout", [dict(gmis_per_gpu=1), dict(gmis_per_gpu=2), dict(decoupled=1, gmi_backend=1)])
def test_nccl_allreduce_in_iteration_graph(cuda, monkeypatch, layout):
    """The cross-GPU gradient all-reduce (ncclAllReduce on the update stream, captured in the
    iteration's CUDA graph) exercised on a one-GPU box through a one-rank communicator
    (GMI_FORCE_NCCL=1): the sum over one rank is the identity, so three iterations (eager, then
    graph replays) must leave the parameters bit-identical to the run without NCCL."""
    from paper_2206_08482_b200.ppo import PpoConfig, Trainer
    cfg = dict(obs_dim=12, act_dim=3, hidden=[64, 64], num_envs=64, **layout)
    plain = Trainer(PpoConfig(**cfg))
    monkeypatch.setenv("GMI_FORCE_NCCL", "1")
    with_nccl = Trainer(PpoConfig(**cfg))
    for _ in range(3):
        plain.iteration()
        with_nccl.iteration()
    assert np.array_equal(plain.get("params").view(np.uint32), with_nccl.get("params").view(np.uint32))


@pytest.mark.parametrize("dims", [(60, 8, [256, 256, 256]), (40, 20, [256, 256])])
def test_pair_weight_gradient_matches_single_cta(cuda, monkeypatch, dims):
    """cuda/gemm_pair.cu (tcgen05 cta_group::2: two SMs form one M = 256 tile, each loading half of
    dPre and half of H) vs the single-CTA split-K kernel on the same minibatch: same slabs, same
    k-block order per output element, so the weight and bias gradients agree to fp32 rounding."""
    S, A, hidden = dims
    g1, g2 = _grad_pair(monkeypatch, "GMI_DW_PAIR", None, dims, envs=1000)
    lay = param_layout(S, A, hidden)
    for key, t in lay.items():
        if not isinstance(key, tuple):
            continue
        for part, n in (("w", t["out_p"] * t["in_p"]), ("b", t["out_p"])):
            a, b = g1[t[part]:t[part] + n], g2[t[part]:t[part] + n]
            assert np.linalg.norm(a - b) <= 1e-6 * (np.linalg.norm(b) + 1e-12), (key, part)


@pytest.mark.parametrize("layout", [dict(gmis_per_gpu=1), dict(gmis_per_gpu=2), dict(decoupled=1, gmi_backend=1)])
def test_minibatch_permutation_indices_are_bit_exact(cuda, layout):
    """The device epoch shuffle gathers rows by the oracle's permutation (Feistel bijection keyed
    by (seed, GMI id, iteration, epoch), ppo_oracle.c): after an iteration the last epoch copy
    holds logp[perm(j)] -- checked bit for bit against the device's own rollout log-probs with
    the oracle's indices, per GMI (integer contract of the north_star)."""
    from golden_util import oracle_perm
    from paper_2206_08482_b200.ppo import PpoConfig, Trainer
    cfg = PpoConfig(obs_dim=12, act_dim=3, hidden=[64, 64], num_envs=64, **layout)
    t = Trainer(cfg)
    for it in range(2):
        t.iteration()
        for gmi in range(cfg.gmis_per_gpu):
            logp = t.get("trained_logp", gmi)
            perm = oracle_perm(cfg.seed, gmi, it, cfg.epochs - 1, logp.size)
            assert np.array_equal(t.get("oldlp_sh", gmi).view(np.uint32), logp[perm].view(np.uint32)), (it, gmi)


@pytest.mark.parametrize("fused_env", [None, ("GMI_ADAM_FUSED", "1")])
@pytest.mark.parametrize("dims", [(60, 8, [256, 256, 256]), (108, 21, [200, 400, 100])])
def test_adam_fused_into_gradient_assembly_is_bit_identical(cuda, monkeypatch, fused_env, dims):
    """One GMI on one GPU: Adam inside the gradient-assembly kernel on the GMI stream (the default
    inline mode, or GMI_ADAM_FUSED=1) vs a separate Adam launch on the update stream
    (GMI_ADAM_INLINE=0) -- same arithmetic per element (quad and block paths of the assembly), so
    three iterations (eager, then graph replays) leave bit-identical parameters."""
    from paper_2206_08482_b200.ppo import PpoConfig, Trainer
    S, A, hidden = dims
    cfg = dict(obs_dim=S, act_dim=A, hidden=hidden, num_envs=256)
    plain = Trainer(PpoConfig(**cfg))
    fused = Trainer(PpoConfig(**cfg))
    for _ in range(3):  # the switches are read when an iteration is recorded (eager, then capture)
        monkeypatch.delenv("GMI_ADAM_FUSED", raising=False)
        monkeypatch.setenv("GMI_ADAM_INLINE", "0")
        plain.iteration()
        monkeypatch.delenv("GMI_ADAM_INLINE", raising=False)
        if fused_env:
            monkeypatch.setenv(*fused_env)
        fused.iteration()
    assert np.array_equal(plain.get("params").view(np.uint32), fused.get("params").view(np.uint32))


@pytest.mark.parametrize("envs", [1536, 4096])
def test_chained_forward_is_bit_identical(cuda, monkeypatch, envs):
    """GemmParams::chain (all hidden forward layers of both nets in one weight-stationary launch,
    each CTA carrying its row tiles through the layers) vs one launch per layer (GMI_FWD_CHAIN=0):
    same tiles, same MMA K order, same epilogue, so two iterations leave bit-identical parameters.
    1536 envs gives CTAs with one and with two row tiles per layer, 4096 the bench's three / four."""
    from paper_2206_08482_b200.ppo import PpoConfig, Trainer
    cfg = dict(obs_dim=60, act_dim=8, hidden=[256, 256, 256], num_envs=envs)
    chained = Trainer(PpoConfig(**cfg))
    monkeypatch.setenv("GMI_FWD_CHAIN", "0")
    plain = Trainer(PpoConfig(**cfg))
    for _ in range(2):
        a, b = chained.iteration(), plain.iteration()
        assert a.kernel_launches < b.kernel_launches  # the chained launch really ran
    assert np.array_equal(chained.get("params").view(np.uint32), plain.get("params").view(np.uint32))
