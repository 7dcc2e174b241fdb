"""Pin the PPO restatement (oracle/ppo_oracle.c) before trusting it as the GPU checker.

The reference has no PPO arithmetic, so the oracle is pinned against independent
implementations: Random123 Philox4x32-10 known-answer vectors, torch's bf16 rounding,
torch float64 autograd for the actor-critic MLP + clipped PPO loss, torch.optim.Adam, a
textbook GAE, and the reference's own contracts (parameter counts workload.hpp:95-100,
env partition reduction.hpp:164-166).
"""
import ctypes as C

import numpy as np
import pytest

from golden_util import PpoOracle, make_cfg, param_layout, ppo_lib

torch = pytest.importorskip("torch")


def philox(k0, k1, ctr):
    out = (C.c_uint32 * 4)()
    ppo_lib().ppo_philox(k0, k1, (C.c_uint32 * 4)(*ctr), out)
    return list(out)


def test_philox_known_answers():
    # Random123 kat_vectors, philox4x32_10
    assert philox(0, 0, [0, 0, 0, 0]) == [0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8]
    assert philox(0xFFFFFFFF, 0xFFFFFFFF, [0xFFFFFFFF] * 4) == [0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD]
    assert philox(0xA4093822, 0x299F31D0, [0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344]) == \
        [0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1]


@pytest.mark.parametrize("n", [1, 2, 3, 7, 64, 100, 1000, 4096, 131072, 6000])
def test_permutation_is_a_bijection(n):
    keys = (C.c_uint32 * 4)(0x12345678, 0x9ABCDEF0, 0x0F0F0F0F, 0xDEADBEEF)
    perm = [ppo_lib().ppo_perm_index(j, n, keys) for j in range(n)]
    assert sorted(perm) == list(range(n))
    if n > 8:
        assert perm != list(range(n))


def test_bf16_rounding_matches_torch():
    rng = np.random.default_rng(0)
    x = np.concatenate([rng.standard_normal(20000).astype(np.float32) * 10 ** rng.uniform(-8, 8, 20000).astype(np.float32),
                        np.array([0.0, -0.0, 1.0, 65504.0, 1e-40, 3.3895314e38], dtype=np.float32)])
    ours = np.array([ppo_lib().ppo_bf16_round(float(v)) for v in x], dtype=np.float32)
    theirs = torch.from_numpy(x).bfloat16().float().numpy()
    assert np.array_equal(ours.view(np.uint32), theirs.view(np.uint32))


@pytest.mark.parametrize("bench,dims", [("AT", [60, 256, 128, 64, 8]), ("HM", [108, 200, 400, 100, 21]),
                                        ("SH", [211, 512, 512, 512, 256, 20])])
def test_real_parameter_count_matches_reference_catalog(bench, dims):
    from paper_2206_08482_b200 import gmux as G
    lay = param_layout(dims[0], dims[-1], dims[1:-1])
    real = sum(v["out"] * v["inp"] + v["out"] for k, v in lay.items() if isinstance(k, tuple))
    assert real == G.policy_value_param_count(dims)
    o = PpoOracle(make_cfg(dims[0], dims[-1], dims[1:-1], 8))
    assert o.P == lay["P"]


def _torch_nets(flat, lay, L):
    nets = []
    for n in range(2):
        layers = []
        for l in range(L + 1):
            t = lay[(n, l)]
            W = torch.tensor(flat[t["w"]:t["w"] + t["out_p"] * t["in_p"]].reshape(t["out_p"], t["in_p"])[:t["out"], :t["inp"]],
                             dtype=torch.float64, requires_grad=True)
            b = torch.tensor(flat[t["b"]:t["b"] + t["out"]], dtype=torch.float64, requires_grad=True)
            layers.append((W, b))
        nets.append(layers)
    log_std = torch.tensor(flat[lay["log_std"]:lay["log_std"] + lay[(0, L)]["out"]], dtype=torch.float64,
                           requires_grad=True)
    return nets, log_std


def _torch_loss(nets, log_std, X, act, oldlp, adv, ret, clip=0.2, vf=1.0, ent=0.0):
    elu = torch.nn.functional.elu

    def fwd(layers, x):
        for W, b in layers[:-1]:
            x = elu(x @ W.T + b)
        W, b = layers[-1]
        return x @ W.T + b

    mu = fwd(nets[0], X)
    v = fwd(nets[1], X)[:, 0]
    dist = torch.distributions.Normal(mu, log_std.exp())
    lp = dist.log_prob(act).sum(-1)
    ratio = torch.exp(lp - oldlp)
    s1, s2 = ratio * adv, torch.clamp(ratio, 1 - clip, 1 + clip) * adv
    lpi = -torch.min(s1, s2).mean()
    lv = 0.5 * vf * ((v - ret) ** 2).mean()
    entropy = dist.entropy().sum(-1).mean()
    return lpi + lv - ent * entropy, lpi, lv


@pytest.mark.parametrize("dims,B", [([12, 64, 32, 3], 96), ([60, 64, 64, 8], 128), ([23, 96, 64, 64, 9], 64)])
def test_minibatch_gradient_matches_torch_autograd(dims, B):
    S, A, hidden = dims[0], dims[-1], dims[1:-1]
    o = PpoOracle(make_cfg(S, A, hidden, 16, exact_fp32=1, ent_coef=0.01))
    lay = param_layout(S, A, hidden)
    flat = o.get("params").astype(np.float64)
    rng = np.random.default_rng(B)
    flat[lay["log_std"]:lay["log_std"] + A] = rng.uniform(-0.5, 0.2, A)
    o.set("params", flat.astype(np.float32))
    flat = o.get("params").astype(np.float64)
    X = rng.uniform(-1, 1, (B, S)).astype(np.float32)
    act = rng.standard_normal((B, A)).astype(np.float32)
    oldlp = (rng.standard_normal(B) - 5).astype(np.float32)
    adv = rng.standard_normal(B).astype(np.float32)
    ret = rng.standard_normal(B).astype(np.float32)
    grad, stats = o.minibatch(X, act, oldlp, adv, ret)

    nets, log_std = _torch_nets(flat, lay, len(hidden))
    T = lambda a: torch.tensor(a, dtype=torch.float64)
    loss, lpi, lv = _torch_loss(nets, log_std, T(X), T(act), T(oldlp), T(adv), T(ret), ent=0.01)
    loss.backward()
    assert stats[0] == pytest.approx(lpi.item(), rel=1e-4, abs=1e-6)
    assert stats[1] == pytest.approx(lv.item(), rel=1e-4, abs=1e-6)
    for n in range(2):
        for l, (W, b) in enumerate(nets[n]):
            t = lay[(n, l)]
            gw = grad[t["w"]:t["w"] + t["out_p"] * t["in_p"]].reshape(t["out_p"], t["in_p"])
            np.testing.assert_allclose(gw[:t["out"], :t["inp"]], W.grad.numpy(), rtol=2e-4, atol=2e-6)
            assert not gw[t["out"]:, :].any() and not gw[:, t["inp"]:].any()  # padding stays zero
            np.testing.assert_allclose(grad[t["b"]:t["b"] + t["out"]], b.grad.numpy(), rtol=2e-4, atol=2e-6)
    np.testing.assert_allclose(grad[lay["log_std"]:lay["log_std"] + A], log_std.grad.numpy(), rtol=2e-4, atol=2e-6)


def test_adam_matches_torch_optim():
    o = PpoOracle(make_cfg(12, 3, [32], 8, lr=1e-3))
    p0 = o.get("params").copy()
    rng = np.random.default_rng(1)
    param = torch.tensor(p0, dtype=torch.float32, requires_grad=True)
    opt = torch.optim.Adam([param], lr=1e-3, betas=(0.9, 0.999), eps=1e-8)
    for step in range(5):
        g = rng.standard_normal(p0.size).astype(np.float32) * 0.01
        o.adam(g)  # one GMI: grad_sum == grad
        param.grad = torch.from_numpy(g.copy())
        opt.step()
    np.testing.assert_allclose(o.get("params"), param.detach().numpy(), rtol=1e-6, atol=1e-7)


def test_gae_matches_textbook_recursion():
    o = PpoOracle(make_cfg(12, 3, [32, 32], 40, horizon=32))
    o.rollout()
    N, T = 40, 32
    rew, val = o.get("rew").reshape(T, N).astype(np.float64), o.get("val").reshape(T + 1, N).astype(np.float64)
    done = o.get("done").reshape(T, N).astype(np.float64)
    adv = np.zeros((T, N))
    last = np.zeros(N)
    for t in reversed(range(T)):
        nt = 1.0 - done[t]
        delta = rew[t] + 0.99 * val[t + 1] * nt - val[t]
        last = delta + 0.99 * 0.95 * nt * last
        adv[t] = last
    np.testing.assert_allclose(o.get("adv").reshape(T, N), adv, rtol=1e-5, atol=1e-5)
    np.testing.assert_allclose(o.get("ret").reshape(T, N), adv + val[:T], rtol=1e-5, atol=1e-5)


def test_reset_masks_follow_integer_episode_clock():
    """done[t][e] is a pure integer function of the per-env episode clock (bit-exact)."""
    o = PpoOracle(make_cfg(12, 3, [32], 50, horizon=32))
    ep_len0, ep_step0 = o.get("ep_len").copy(), o.get("ep_step").copy()
    o.rollout()
    done = o.get("done").reshape(32, 50)
    step = ep_step0.copy()
    count = np.zeros(50, dtype=np.int32)
    for t in range(32):
        d = (step + 1 >= ep_len0)
        assert np.array_equal(done[t].astype(bool), d)
        step = np.where(d, 0, step + 1)
        count += d
    assert np.array_equal(o.get("ep_count"), count)
    assert ((16 <= ep_len0) & (ep_len0 < 64)).all()


def test_env_partition_makes_rollouts_layout_invariant():
    """Envs are partitioned over GMIs by [N*c/n, N*(c+1)/n) (reduction.hpp:164-166) and all
    randomness is keyed by the global env id, so the first rollout is identical bit-for-bit
    under 1 GMI or 2 GPUs x 2 GMIs."""
    one = PpoOracle(make_cfg(12, 3, [32], 50))
    four = PpoOracle(make_cfg(12, 3, [32], 50, num_gpus=2, gmis_per_gpu=2))
    one.rollout()
    four.rollout()
    rew1 = one.get("rew").reshape(32, 50)
    parts = [four.get("rew", c).reshape(32, -1) for c in range(4)]
    assert [p.shape[1] for p in parts] == [12, 13, 12, 13]
    assert np.array_equal(np.concatenate(parts, axis=1), rew1)
    assert np.array_equal(np.concatenate([four.get("done", c).reshape(32, -1) for c in range(4)], axis=1),
                          one.get("done").reshape(32, 50))


def test_full_iteration_runs_and_learns_something():
    o = PpoOracle(make_cfg(12, 3, [32, 32], 64, num_gpus=1, gmis_per_gpu=2))
    p0 = o.get("params").copy()
    s = o.iteration()
    assert s.env_steps == 64 * 32
    assert np.isfinite([s.policy_loss, s.value_loss, s.approx_kl]).all()
    assert not np.array_equal(o.get("params"), p0)


def test_decoupled_first_iteration_equals_synchronous():
    """Decoupled mode (serving GMI + trainer GMI, one-iteration policy lag): iteration 0 trains
    on rollout 0, produced with theta_0 exactly as in the synchronous iteration, so the
    parameters after it are bit-identical; from iteration 1 on the experience is one policy
    version behind and the trajectories diverge."""
    sync = PpoOracle(make_cfg(12, 3, [32, 32], 64))
    dec = PpoOracle(make_cfg(12, 3, [32, 32], 64))
    s0 = sync.iteration()
    d0 = dec.iteration_decoupled()
    assert np.array_equal(sync.get("params").view(np.uint32), dec.get("params").view(np.uint32))
    assert s0.mean_reward == d0.mean_reward and d0.env_steps == 64 * 32
    sync.iteration()
    dec.iteration_decoupled()
    assert not np.array_equal(sync.get("params"), dec.get("params"))


def test_decoupled_rollout_uses_the_lagged_policy():
    """Rollout i+1 is produced with theta_i: replaying it with a synchronous handle whose
    parameters are set to theta_i (and whose env state is rollout i's) reproduces it."""
    dec = PpoOracle(make_cfg(12, 3, [32], 64))
    dec.iteration_decoupled()        # trains rollout 0 -> theta_1; produces rollout 1 with theta_0
    # a synchronous handle at iteration 1 (env state after rollout 0) whose parameters are
    # reset to theta_0 produces the same rollout 1
    ref2 = PpoOracle(make_cfg(12, 3, [32], 64))
    theta0 = ref2.get("params").copy()
    ref2.iteration()                 # env state after rollout 0, iteration counter 1
    ref2.set("params", theta0)
    ref2.rollout()                   # rollout 1 with theta_0
    for what in ("rew", "act", "logp", "done"):
        assert np.array_equal(dec.get(what), ref2.get(what)), what


def _bf(x):
    return x.to(torch.bfloat16).to(x.dtype)


class _RoundFwd(torch.autograd.Function):
    """bf16 rounding of a forward value (operands the device stores in bf16); identity backward."""

    @staticmethod
    def forward(ctx, x):
        return _bf(x)

    @staticmethod
    def backward(ctx, g):
        return g


class _RoundBwd(torch.autograd.Function):
    """Identity forward; bf16 rounding of the incoming gradient (head output grads G_pi / G_v)."""

    @staticmethod
    def forward(ctx, x):
        return x.clone()

    @staticmethod
    def backward(ctx, g):
        return _bf(g)


class _EluBf16(torch.autograd.Function):
    """Hidden activation as the device computes it: H = bf16(elu(pre)); dPre = bf16(dH * elu'(H)),
    elu'(H) = H > 0 ? 1 : H + 1 (from the stored bf16 output)."""

    @staticmethod
    def forward(ctx, pre):
        h = _bf(torch.nn.functional.elu(pre))
        ctx.save_for_backward(h)
        return h

    @staticmethod
    def backward(ctx, g):
        (h,) = ctx.saved_tensors
        return _bf(g * torch.where(h > 0, torch.ones_like(h), h + 1))


@pytest.mark.parametrize("dims,B", [([12, 64, 32, 3], 96), ([60, 64, 64, 8], 128), ([23, 96, 64, 64, 9], 64)])
def test_bf16_mode_gradient_matches_torch_with_the_same_rounding_points(dims, B):
    """The default (bf16) oracle mode -- the GPU checker -- against torch float64 autograd with bf16
    rounding at exactly the device's storage points: observations, every weight matrix, hidden
    activations, pre-activation gradients and head output gradients. Measured agreement ~2e-8
    relative (float vs double accumulation before a rounding point); bound 1e-5."""
    S, A, hidden = dims[0], dims[-1], dims[1:-1]
    o = PpoOracle(make_cfg(S, A, hidden, 16, ent_coef=0.01))
    lay = param_layout(S, A, hidden)
    flat = o.get("params").astype(np.float64)
    rng = np.random.default_rng(B + 1)
    # observations are stored in bf16 (rollout buffer) before they reach the update
    X = torch.from_numpy(rng.uniform(-1, 1, (B, S)).astype(np.float32)).bfloat16().float().numpy()
    act = rng.standard_normal((B, A)).astype(np.float32)
    oldlp = (rng.standard_normal(B) - 5).astype(np.float32)
    adv = rng.standard_normal(B).astype(np.float32)
    ret = rng.standard_normal(B).astype(np.float32)
    grad, stats = o.minibatch(X, act, oldlp, adv, ret)

    nets, log_std = _torch_nets(flat, lay, len(hidden))
    T = lambda a: torch.tensor(a, dtype=torch.float64)

    def fwd(layers, x):
        x = _RoundFwd.apply(x)
        for W, b in layers[:-1]:
            x = _EluBf16.apply(x @ _RoundFwd.apply(W).T + b)
        W, b = layers[-1]
        return _RoundBwd.apply(x @ _RoundFwd.apply(W).T) + b  # bias gradient from the unrounded G

    mu = fwd(nets[0], T(X))
    v = fwd(nets[1], T(X))[:, 0]
    dist = torch.distributions.Normal(mu, log_std.exp())
    lp = dist.log_prob(T(act)).sum(-1)
    ratio = torch.exp(lp - T(oldlp))
    s1, s2 = ratio * T(adv), torch.clamp(ratio, 0.8, 1.2) * T(adv)
    loss = -torch.min(s1, s2).mean() + 0.5 * ((v - T(ret)) ** 2).mean() - 0.01 * dist.entropy().sum(-1).mean()
    loss.backward()
    for n in range(2):
        for l, (W, b) in enumerate(nets[n]):
            t = lay[(n, l)]
            gw = grad[t["w"]:t["w"] + t["out_p"] * t["in_p"]].reshape(t["out_p"], t["in_p"])[:t["out"], :t["inp"]]
            ref = W.grad.numpy()
            assert np.linalg.norm(gw - ref) <= 1e-5 * np.linalg.norm(ref), (n, l)
            gb, rb = grad[t["b"]:t["b"] + t["out"]], b.grad.numpy()
            assert np.linalg.norm(gb - rb) <= 1e-5 * np.linalg.norm(rb) + 1e-9, (n, l, "b")
    gl = grad[lay["log_std"]:lay["log_std"] + A]
    np.testing.assert_allclose(gl, log_std.grad.numpy(), rtol=1e-5, atol=1e-7)
