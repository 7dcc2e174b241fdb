"""Python handle over libgmi's B200 PPO trainer (gmi_ppo_* in include/gmi.h).

One ``Trainer`` drives one GPU of a data-parallel job.  Everything runs in libgmi.so
(tcgen05 GEMMs, env / head / GAE / Adam kernels, K1 reduction, NCCL); this module only
marshals configuration and host copies.  There is no CPU path.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

from . import _lib as L

MAX_HIDDEN = 8


class PpoConfigT(C.Structure):
    _fields_ = [("obs_dim", C.c_int), ("act_dim", C.c_int), ("num_hidden", C.c_int),
                ("hidden", C.c_int * MAX_HIDDEN), ("num_envs", C.c_int), ("horizon", C.c_int),
                ("epochs", C.c_int), ("minibatches", C.c_int), ("gamma", C.c_float),
                ("lam", C.c_float), ("clip", C.c_float), ("lr", C.c_float), ("beta1", C.c_float),
                ("beta2", C.c_float), ("adam_eps", C.c_float), ("vf_coef", C.c_float),
                ("ent_coef", C.c_float), ("seed", C.c_ulonglong), ("num_gpus", C.c_int),
                ("gmis_per_gpu", C.c_int), ("rank", C.c_int), ("device", C.c_int),
                ("gmi_backend", C.c_int), ("sm_per_gmi", C.c_int), ("use_graph", C.c_int),
                ("instrument", C.c_int), ("decoupled", C.c_int), ("serving_sms", C.c_int),
                ("comm", C.c_int)]


PPO_PHASES = 20  # GMI_PPO_PHASES


class PhaseT(C.Structure):
    _fields_ = [("ms", C.c_double), ("flop", C.c_double), ("bytes", C.c_double), ("launches", C.c_int)]


class PpoStatsT(C.Structure):
    _fields_ = [("policy_loss", C.c_double), ("value_loss", C.c_double), ("approx_kl", C.c_double),
                ("clip_frac", C.c_double), ("mean_reward", C.c_double), ("env_steps", C.c_longlong),
                ("gemm_ms", C.c_double), ("gemm_flop", C.c_double), ("gemm_launches", C.c_int),
                ("kernel_launches", C.c_int), ("gemm_bytes", C.c_double)]


_PROTOS = {
    "gmi_ppo_config_defaults": (None, [C.POINTER(PpoConfigT)]),
    "gmi_ppo_create": (C.c_int, [C.POINTER(PpoConfigT), C.c_void_p, C.POINTER(C.c_void_p)]),
    "gmi_ppo_free": (None, [C.c_void_p]),
    "gmi_nccl_unique_id": (C.c_int, [C.c_void_p]),
    "gmi_ppo_iteration": (C.c_int, [C.c_void_p, C.POINTER(PpoStatsT)]),
    "gmi_ppo_iteration_async": (C.c_int, [C.c_void_p]),
    "gmi_ppo_synchronize": (C.c_int, [C.c_void_p, C.POINTER(PpoStatsT)]),
    "gmi_ppo_rollout": (C.c_int, [C.c_void_p]),
    "gmi_ppo_comm_handle": (C.c_int, [C.c_void_p, C.c_void_p]),
    "gmi_resize": (C.c_int, [C.c_void_p, C.c_int, C.POINTER(C.c_int), C.c_int]),
    "gmi_ppo_tune_shares": (C.c_int, [C.c_void_p, C.POINTER(C.c_int), C.c_int, C.c_int, C.POINTER(C.c_int),
                                      C.POINTER(C.c_double)]),
    "gmi_ppo_comm_attach": (C.c_int, [C.c_void_p, C.c_void_p]),
    "gmi_ppo_comm_connect": (C.c_int, [C.POINTER(C.c_void_p), C.c_int]),
    "gmi_ppo_link_handle": (C.c_int, [C.c_void_p, C.c_void_p]),
    "gmi_ppo_link_attach": (C.c_int, [C.c_void_p, C.c_void_p]),
    "gmi_ppo_link_connect": (C.c_int, [C.c_void_p, C.c_void_p]),
    "gmi_ppo_minibatch_grad": (C.c_int, [C.c_void_p, C.c_int] + [C.POINTER(C.c_float)] * 5 +
                               [C.c_int, C.POINTER(C.c_float)]),
    "gmi_ppo_get": (C.c_int, [C.c_void_p, C.c_char_p, C.c_int, C.c_void_p, C.POINTER(C.c_longlong)]),
    "gmi_ppo_set": (C.c_int, [C.c_void_p, C.c_char_p, C.c_int, C.c_void_p, C.c_longlong]),
    "gmi_ppo_param_count": (C.c_int, [C.c_void_p, C.POINTER(C.c_longlong), C.POINTER(C.c_longlong)]),
    "gmi_ppo_stream": (C.c_int, [C.c_void_p, C.c_int, C.POINTER(C.c_void_p)]),
    "gmi_ppo_phase_name": (C.c_char_p, [C.c_int]),
    "gmi_ppo_profile": (C.c_int, [C.c_void_p, C.c_void_p]),
    "gmi_ppo_set_instrument": (C.c_int, [C.c_void_p, C.c_int]),
    "gmi_ppo_unit_busy": (C.c_int, [C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_int), C.c_int,
                                    C.POINTER(C.c_int)]),
}
L.PROTOTYPES.update(_PROTOS)
if L._lib is not None:  # library already loaded: bind the late prototypes
    for _n, (_r, _a) in _PROTOS.items():
        getattr(L._lib, _n).restype, getattr(L._lib, _n).argtypes = _r, _a


@dataclass
class PpoConfig:
    obs_dim: int = 60
    act_dim: int = 8
    hidden: list = field(default_factory=lambda: [256, 256, 256])
    num_envs: int = 4096
    horizon: int = 32
    epochs: int = 4
    minibatches: int = 4
    gamma: float = 0.99
    lam: float = 0.95
    clip: float = 0.2
    lr: float = 3e-4
    beta1: float = 0.9
    beta2: float = 0.999
    adam_eps: float = 1e-8
    vf_coef: float = 1.0
    ent_coef: float = 0.0
    seed: int = 20240811
    num_gpus: int = 1
    gmis_per_gpu: int = 1
    rank: int = 0
    device: int = 0
    gmi_backend: int = 0
    sm_per_gmi: int = 0
    use_graph: int = 1
    instrument: int = 0
    decoupled: int = 0
    serving_sms: int = 0
    comm: int = 0  # num_gpus > 1: 0 NCCL all-reduce, 1 peer exchange (fused reduce-scatter/Adam/all-gather)

    def to_c(self) -> PpoConfigT:
        c = PpoConfigT()
        L.lib().gmi_ppo_config_defaults(C.byref(c))
        for k, v in self.__dict__.items():
            if k == "hidden":
                c.num_hidden = len(v)
                for i, h in enumerate(v):
                    c.hidden[i] = h
            else:
                setattr(c, k, v)
        return c

    @staticmethod
    def from_benchmark(name: str, num_envs: int, hidden=None, **kw) -> "PpoConfig":
        """Shapes from the reference catalog (workload.hpp:126-134) via libgmi."""
        from . import gmux
        w = gmux.load_benchmark(name)
        dims = w.policy_dims
        return PpoConfig(obs_dim=dims[0], act_dim=dims[-1], hidden=list(hidden or dims[1:-1]),
                         num_envs=num_envs, horizon=w.steps_per_train, **kw)

    @staticmethod
    def from_config_file(path: str, **kw) -> "PpoConfig":
        """proj/configs schema + the B200 [ppo] section (ignored by the reference parser)."""
        from . import gmux
        cfg = gmux.load_config(path)
        w = gmux.workload_from_config(cfg)
        model = gmux.model_from_config(cfg)
        topo = gmux.topology_from_config(cfg)
        dims = w.policy_dims
        hidden = cfg.get("ppo", "hidden")
        out = PpoConfig(obs_dim=dims[0], act_dim=dims[-1],
                        hidden=[int(h) for h in hidden.split(",")] if hidden else dims[1:-1],
                        num_envs=int(cfg.get("ppo", "num_envs") or 4096),
                        horizon=int(cfg.get("ppo", "horizon") or w.steps_per_train),
                        epochs=int(cfg.get("ppo", "epochs") or 4),
                        minibatches=int(cfg.get("ppo", "minibatches") or 4),
                        gmis_per_gpu=model.gmis_per_gpu, num_gpus=max(1, len(topo.gpus)),
                        decoupled=int(cfg.get("ppo", "decoupled") or 0),
                        serving_sms=int(cfg.get("ppo", "serving_sms") or 0))
        backend = cfg.get("ppo", "gmi_backend")
        if out.decoupled:  # [model] gmis_per_gpu counts all GMIs; the trainer side is one per GPU
            out.gmis_per_gpu = 1
            out.gmi_backend = int(backend or 1)
        else:
            # The topology's MPS partitions of the first GPU are the GMIs (topology.hpp:72-88): on
            # B200 each share is realised as a green context of whole 8-SM groups (gmi_green_sms).
            first = min((g.id for g in topo.gpus), default=0)
            parts = [p for p in topo.partitions if p.gpu_id == first]
            partitioned = any(p.backend == gmux.Backend.MPS and p.sm_share < 1.0 for p in parts)
            out.gmi_backend = int(backend) if backend is not None else (1 if partitioned else 0)
            if out.gmi_backend == 1 and parts:
                if len(parts) != out.gmis_per_gpu:
                    raise gmux.ConfigError(f"{path}: [model] gmis_per_gpu = {out.gmis_per_gpu} but GPU {first} "
                                           f"has {len(parts)} gmi partitions")
                shares = sorted({round(p.sm_share, 9) for p in parts})
                if len(shares) != 1:
                    raise gmux.ConfigError(f"{path}: unequal MPS shares {shares} cannot be realised as equal "
                                           "green-context GMIs")
                out.sm_per_gmi = gmux.green_sms(shares[0])
                if out.sm_per_gmi < 8 or out.sm_per_gmi * len(parts) > 148:
                    raise gmux.ConfigError(f"{path}: share {shares[0]} x {len(parts)} GMIs is not realisable "
                                           "on a 148-SM B200 in 8-SM groups")
        for k, v in kw.items():
            setattr(out, k, v)
        return out


def nccl_unique_id() -> bytes:
    buf = (C.c_char * 128)()
    L.check(L.lib().gmi_nccl_unique_id(buf))
    return bytes(buf)


@dataclass
class IterationStats:
    policy_loss: float
    value_loss: float
    approx_kl: float
    clip_frac: float
    mean_reward: float
    env_steps: int
    gemm_ms: float
    gemm_flop: float
    gemm_launches: int
    kernel_launches: int
    gemm_bytes: float = 0.0


_DT = {"done": np.uint8, "ep_step": np.int32, "ep_len": np.int32, "ep_count": np.int32,
       "rollout_trace": np.int64, "train_fwd_trace": np.int64, "gemm_trace": np.int64, "head_trace": np.int64}


class Trainer:
    def __init__(self, cfg: PpoConfig, nccl_id: bytes | None = None):
        self.cfg = cfg
        self._c = cfg.to_c()
        h = C.c_void_p()
        idbuf = C.create_string_buffer(nccl_id, 128) if nccl_id else None
        L.check(L.lib().gmi_ppo_create(C.byref(self._c), idbuf, C.byref(h)))
        self._h = h
        p, r = C.c_longlong(), C.c_longlong()
        L.check(L.lib().gmi_ppo_param_count(h, C.byref(p), C.byref(r)))
        self.param_count, self.real_param_count = p.value, r.value

    def close(self):
        if getattr(self, "_h", None) and L is not None:
            L.lib().gmi_ppo_free(self._h)
            self._h = None

    __del__ = close

    @staticmethod
    def _stats(s: PpoStatsT) -> IterationStats:
        return IterationStats(s.policy_loss, s.value_loss, s.approx_kl, s.clip_frac, s.mean_reward,
                              s.env_steps, s.gemm_ms, s.gemm_flop, s.gemm_launches, s.kernel_launches,
                              s.gemm_bytes)

    def iteration(self) -> IterationStats:
        s = PpoStatsT()
        L.check(L.lib().gmi_ppo_iteration(self._h, C.byref(s)))
        return self._stats(s)

    def iteration_async(self) -> None:
        L.check(L.lib().gmi_ppo_iteration_async(self._h))

    def synchronize(self) -> IterationStats:
        s = PpoStatsT()
        L.check(L.lib().gmi_ppo_synchronize(self._h, C.byref(s)))
        return self._stats(s)

    def rollout(self) -> None:
        L.check(L.lib().gmi_ppo_rollout(self._h))

    def resize(self, sm_counts: list) -> None:
        """Re-split this GPU's green-context partitions (gmi_resize); same GMI count. The GMI
        streams (and, in the one-GPU decoupled layout, the update stream) are recreated in the new
        partitions: re-read stream() afterwards."""
        arr = (C.c_int * len(sm_counts))(*sm_counts)
        L.check(L.lib().gmi_resize(self._h, self.cfg.rank, arr, len(sm_counts)))

    def tune_shares(self, candidates: list, iters: int = 3):
        """Measured per-role SM-share retuning (gmi_ppo_tune_shares): returns (best index,
        env-steps/s per candidate); the trainer is left at the best split (streams recreated, as
        for resize())."""
        flat = [x for c in candidates for x in c]
        arr = (C.c_int * len(flat))(*flat)
        out = (C.c_double * len(candidates))()
        best = C.c_int()
        L.check(L.lib().gmi_ppo_tune_shares(self._h, arr, len(candidates), iters, C.byref(best), out))
        return best.value, list(out)

    def comm_handle(self) -> bytes:
        """64-byte CUDA IPC handle of this rank's exchange window (cfg.comm = 1)."""
        buf = (C.c_char * 64)()
        L.check(L.lib().gmi_ppo_comm_handle(self._h, buf))
        return bytes(buf)

    def comm_attach(self, handles: list) -> None:
        """Wire the peer exchange from every rank's comm_handle(), in rank order."""
        blob = b"".join(handles)
        L.check(L.lib().gmi_ppo_comm_attach(self._h, C.create_string_buffer(blob, len(blob))))

    @staticmethod
    def comm_connect(trainers: list) -> None:
        """Wire the peer exchange of trainers living in this process (trainers[r] = rank r)."""
        arr = (C.c_void_p * len(trainers))(*[t._h.value for t in trainers])
        L.check(L.lib().gmi_ppo_comm_connect(arr, len(trainers)))

    def link_handle(self) -> bytes:
        """64-byte CUDA IPC handle of this rank's experience-link window (decoupled = 2)."""
        buf = (C.c_char * 64)()
        L.check(L.lib().gmi_ppo_link_handle(self._h, buf))
        return bytes(buf)

    def link_attach(self, peer_handle: bytes) -> None:
        """Wire the AsyncDecoupled pair from the partner's link_handle() (serving rank s <->
        trainer rank num_gpus / 2 + s)."""
        L.check(L.lib().gmi_ppo_link_attach(self._h, C.create_string_buffer(peer_handle, 64)))

    @staticmethod
    def link_connect(serving: "Trainer", trainer: "Trainer") -> None:
        """Wire an AsyncDecoupled pair living in this process (distinct devices)."""
        L.check(L.lib().gmi_ppo_link_connect(serving._h, trainer._h))

    def stream(self, gmi: int = -1) -> int:
        s = C.c_void_p()
        L.check(L.lib().gmi_ppo_stream(self._h, gmi, C.byref(s)))
        return s.value or 0

    def set_instrument(self, on: bool) -> None:
        L.check(L.lib().gmi_ppo_set_instrument(self._h, int(bool(on))))

    def profile(self) -> dict:
        """Per-phase device time of the last iteration run with instrumentation on:
        {phase: {"ms", "flop", "bytes", "launches"}} (GMI 0 stream + update stream)."""
        arr = (PhaseT * PPO_PHASES)()
        L.check(L.lib().gmi_ppo_profile(self._h, arr))
        return {L.lib().gmi_ppo_phase_name(i).decode(): {"ms": a.ms, "flop": a.flop, "bytes": a.bytes,
                                                        "launches": a.launches}
                for i, a in enumerate(arr)}

    def unit_busy(self) -> list:
        """[(busy_ms, sms)] per execution unit of the last instrumented iteration: decoupled ->
        serving GMI, trainer GMI; else the local GMIs; last = the update stream."""
        n = C.c_int()
        L.check(L.lib().gmi_ppo_unit_busy(self._h, None, None, 0, C.byref(n)))
        busy, sms = (C.c_double * n.value)(), (C.c_int * n.value)()
        L.check(L.lib().gmi_ppo_unit_busy(self._h, busy, sms, n.value, C.byref(n)))
        return [(busy[i], sms[i]) for i in range(n.value)]

    def get(self, what: str, gmi: int = 0) -> np.ndarray:
        n = C.c_longlong()
        L.check(L.lib().gmi_ppo_get(self._h, what.encode(), gmi, None, C.byref(n)))
        out = np.empty(n.value, dtype=_DT.get(what, np.float32))
        L.check(L.lib().gmi_ppo_get(self._h, what.encode(), gmi, out.ctypes.data, C.byref(n)))
        return out

    def set(self, what: str, arr, gmi: int = 0) -> None:
        a = np.ascontiguousarray(arr, dtype=_DT.get(what, np.float32))
        L.check(L.lib().gmi_ppo_set(self._h, what.encode(), gmi, a.ctypes.data, a.size))

    def minibatch_grad(self, X, act, oldlp, adv, ret, gmi: int = 0) -> np.ndarray:
        fp = C.POINTER(C.c_float)
        arrs = [np.ascontiguousarray(a, dtype=np.float32) for a in (X, act, oldlp, adv, ret)]
        grad = np.zeros(self.param_count, dtype=np.float32)
        L.check(L.lib().gmi_ppo_minibatch_grad(self._h, gmi, *[a.ctypes.data_as(fp) for a in arrs],
                                               len(arrs[2]), grad.ctypes.data_as(fp)))
        return grad
