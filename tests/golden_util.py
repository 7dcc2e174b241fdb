"""Shared helpers for parity tests: golden-buffer generation and oracle loading.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may load oracle/.
"""
from __future__ import annotations

import ctypes as C
import hashlib
import json
import os

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
ORACLE_DIR = os.path.join(ROOT, "oracle", "_ref")


def cases(name: str):
    with open(os.path.join(GOLDEN, f"ref_{name}.json")) as f:
        return json.load(f)["cases"]


def buffer_values(kind: str, seed: int, gid: int, length: int) -> np.ndarray:
    """numpy mirror of buffer_value() in oracle/ref_driver.cpp (bit-identical doubles)."""
    e = np.arange(length, dtype=np.uint64)
    if kind == "cli":
        return 1.0 + 0.001 * gid + 1e-6 * e.astype(np.float64)
    with np.errstate(over="ignore"):
        z = (np.uint64(seed) * np.uint64(0x9E3779B97F4A7C15)
             + np.uint64(gid % (1 << 64)) * np.uint64(0xBF58476D1CE4E5B9)
             + e * np.uint64(0x94D049BB133111EB))
        z = z + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    u = (z >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)
    return 0.1 + 0.9 * u


def f64_digest(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype="<f8").tobytes()).hexdigest()


def layout_arrays(mpl):
    counts = [len(l) for l in mpl]
    ids = [i for l in mpl for i in l]
    return counts, ids


_reduce_oracle = None


def reduce_oracle():
    global _reduce_oracle
    if _reduce_oracle is None:
        path = os.path.join(ORACLE_DIR, "libreduce_oracle.so")
        lib = C.CDLL(path)
        for name in ("oracle_execute_f32", "oracle_execute_f64"):
            fn = getattr(lib, name)
            fn.restype = C.c_int
            fn.argtypes = [C.c_int, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_void_p),
                           C.c_size_t, C.c_void_p]
        _reduce_oracle = lib
    return _reduce_oracle


def oracle_execute(algo: int, mpl, bufs: list[np.ndarray]) -> np.ndarray:
    counts, ids = layout_arrays(mpl)
    dtype = bufs[0].dtype
    length = bufs[0].shape[0]
    out = np.empty(length, dtype=dtype)
    arr = [np.ascontiguousarray(b) for b in bufs]
    ptrs = (C.c_void_p * len(arr))(*[a.ctypes.data for a in arr])
    fn = reduce_oracle().oracle_execute_f64 if dtype == np.float64 else reduce_oracle().oracle_execute_f32
    rc = fn(algo, len(mpl), (C.c_int * len(counts))(*counts), (C.c_int * len(ids))(*ids), ptrs, length,
            out.ctypes.data)
    if rc != 0:
        raise RuntimeError(f"oracle rejected layout (rc={rc})")
    return out


# ------------------------------------------------------------------ PPO oracle (oracle/ppo_oracle.c)
class PpoCfg(C.Structure):
    _fields_ = [("obs_dim", C.c_int), ("act_dim", C.c_int), ("num_hidden", C.c_int),
                ("hidden", C.c_int * 8), ("num_envs", C.c_int), ("horizon", C.c_int),
                ("epochs", C.c_int), ("minibatches", C.c_int), ("gamma", C.c_float),
                ("lam", C.c_float), ("clip", C.c_float), ("lr", C.c_float), ("beta1", C.c_float),
                ("beta2", C.c_float), ("adam_eps", C.c_float), ("vf_coef", C.c_float),
                ("ent_coef", C.c_float), ("seed", C.c_ulonglong), ("num_gpus", C.c_int),
                ("gmis_per_gpu", C.c_int), ("threads", C.c_int), ("exact_fp32", C.c_int)]


class PpoStats(C.Structure):
    _fields_ = [("policy_loss", C.c_double), ("value_loss", C.c_double), ("entropy", C.c_double),
                ("approx_kl", C.c_double), ("clip_frac", C.c_double), ("mean_reward", C.c_double),
                ("env_steps", C.c_longlong)]


PPO_DEFAULTS = dict(horizon=32, epochs=4, minibatches=4, gamma=0.99, lam=0.95, clip=0.2, lr=3e-4,
                    beta1=0.9, beta2=0.999, adam_eps=1e-8, vf_coef=1.0, ent_coef=0.0, seed=20240811,
                    num_gpus=1, gmis_per_gpu=1, threads=0, exact_fp32=0)

_ppo = None


def ppo_lib():
    global _ppo
    if _ppo is None:
        lib = C.CDLL(os.path.join(ORACLE_DIR, "libppo_oracle.so"))
        vp = C.c_void_p
        fp = C.POINTER(C.c_float)
        sig = {
            "ppo_oracle_create": (vp, [C.POINTER(PpoCfg)]),
            "ppo_oracle_free": (None, [vp]),
            "ppo_oracle_iteration": (C.c_int, [vp, C.POINTER(PpoStats)]),
            "ppo_oracle_rollout": (C.c_int, [vp]),
            "ppo_oracle_iteration_decoupled": (C.c_int, [vp, C.POINTER(PpoStats)]),
            "ppo_oracle_minibatch": (C.c_int, [vp, C.c_int, fp, fp, fp, fp, fp, C.c_int, fp,
                                               C.POINTER(C.c_double)]),
            "ppo_oracle_adam": (C.c_int, [vp, fp]),
            "ppo_oracle_param_count": (C.c_longlong, [vp]),
            "ppo_oracle_width": (C.c_int, [vp, C.c_int]),
            "ppo_oracle_get": (C.c_int, [vp, C.c_char_p, C.c_int, vp, C.c_longlong]),
            "ppo_oracle_set": (C.c_int, [vp, C.c_char_p, C.c_int, vp, C.c_longlong]),
            "ppo_philox": (None, [C.c_uint32, C.c_uint32, C.POINTER(C.c_uint32), C.POINTER(C.c_uint32)]),
            "ppo_perm_index": (C.c_uint32, [C.c_uint32, C.c_uint32, C.POINTER(C.c_uint32)]),
            "ppo_oracle_perm": (C.c_int, [C.c_ulonglong, C.c_int, C.c_int, C.c_int, C.c_uint32,
                                          C.POINTER(C.c_uint32)]),
            "ppo_bf16_round": (C.c_float, [C.c_float]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(lib, name)
            fn.restype, fn.argtypes = res, args
        _ppo = lib
    return _ppo


def make_cfg(obs_dim, act_dim, hidden, num_envs, **kw):
    d = dict(PPO_DEFAULTS)
    d.update(kw)
    c = PpoCfg()
    c.obs_dim, c.act_dim, c.num_hidden = obs_dim, act_dim, len(hidden)
    for i, h in enumerate(hidden):
        c.hidden[i] = h
    c.num_envs = num_envs
    for k, v in d.items():
        setattr(c, k, v)
    return c


class PpoOracle:
    """ctypes handle over oracle/ppo_oracle.c (test infrastructure)."""

    DT = {"done": np.uint8, "ep_step": np.int32, "ep_len": np.int32, "ep_count": np.int32}

    def __init__(self, cfg: PpoCfg):
        self.cfg = cfg
        self.h = ppo_lib().ppo_oracle_create(C.byref(cfg))
        if not self.h:
            raise ValueError("oracle rejected config")
        self.P = ppo_lib().ppo_oracle_param_count(self.h)

    def __del__(self):
        if getattr(self, "h", None):
            ppo_lib().ppo_oracle_free(self.h)
            self.h = None

    def get(self, what, gmi=0):
        n = ppo_lib().ppo_oracle_get(self.h, what.encode(), gmi, None, 0)
        if n < 0:
            raise KeyError(what)
        out = np.empty(n, dtype=self.DT.get(what, np.float32))
        ppo_lib().ppo_oracle_get(self.h, what.encode(), gmi, out.ctypes.data, n)
        return out

    def set(self, what, arr, gmi=0):
        arr = np.ascontiguousarray(arr, dtype=self.DT.get(what, np.float32))
        rc = ppo_lib().ppo_oracle_set(self.h, what.encode(), gmi, arr.ctypes.data, arr.size)
        if rc != 0:
            raise ValueError(what)

    def iteration(self):
        s = PpoStats()
        ppo_lib().ppo_oracle_iteration(self.h, C.byref(s))
        return s

    def rollout(self):
        if ppo_lib().ppo_oracle_rollout(self.h) != 0:
            raise RuntimeError("a rollout is already pending: run iteration() to train on it")

    def iteration_decoupled(self):
        s = PpoStats()
        ppo_lib().ppo_oracle_iteration_decoupled(self.h, C.byref(s))
        return s

    def width(self, layer):
        return ppo_lib().ppo_oracle_width(self.h, layer)

    def minibatch(self, X, act, oldlp, adv, ret, gmi=0):
        fp = C.POINTER(C.c_float)
        arrs = [np.ascontiguousarray(a, dtype=np.float32) for a in (X, act, oldlp, adv, ret)]
        grad = np.zeros(self.P, dtype=np.float32)
        stats = (C.c_double * 4)()
        ppo_lib().ppo_oracle_minibatch(self.h, gmi, *[a.ctypes.data_as(fp) for a in arrs], len(oldlp),
                                       grad.ctypes.data_as(fp), stats)
        return grad, list(stats)

    def adam(self, grad_sum):
        g = np.ascontiguousarray(grad_sum, dtype=np.float32)
        ppo_lib().ppo_oracle_adam(self.h, g.ctypes.data_as(C.POINTER(C.c_float)))


def oracle_perm(seed, gmi, iteration, epoch, n):
    out = np.empty(n, dtype=np.uint32)
    ppo_lib().ppo_oracle_perm(seed, gmi, iteration, epoch, n, out.ctypes.data_as(C.POINTER(C.c_uint32)))
    return out


def param_layout(obs_dim, act_dim, hidden):
    """Offsets of the flat parameter vector shared by oracle and device trainer:
    per net (policy, value) per layer (hidden..., head): W [out_p x in_p] then b [out_p],
    each 64-element aligned; widths padded to 32; then log_std [A]."""
    pad = lambda x: (x + 31) // 32 * 32
    al = lambda x: (x + 63) // 64 * 64
    widths = [obs_dim] + list(hidden)
    off, out = 0, {}
    for n in range(2):
        for l in range(len(hidden) + 1):
            fin = widths[l]
            fout = widths[l + 1] if l < len(hidden) else (act_dim if n == 0 else 1)
            fin_p = pad(fin)
            fout_p = pad(fout) if l < len(hidden) else fout
            out[(n, l)] = dict(w=off, out=fout, inp=fin, out_p=fout_p, in_p=fin_p)
            off = al(off + fout_p * fin_p)
            out[(n, l)]["b"] = off
            off = al(off + fout_p)
    out["log_std"] = off
    out["P"] = al(off + act_dim)
    return out
