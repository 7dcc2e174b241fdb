"""Python mirror of the reference's ``namespace gmux`` over libgmi's C-ABI.

Same names, argument meaning and error behaviour as the reference headers
(proj/include/gmux/*.hpp), so parity tests read like the reference's own Catch2 suites.
Exception mapping: ``std::invalid_argument`` -> ``ValueError``; ``MultiStreamError``,
``PlanError``, ``PipelineError``, ``ConfigError`` -> classes below (RuntimeError
subclasses, as in C++).  All logic runs in libgmi.so; this module only marshals.
"""
from __future__ import annotations

import ctypes as C
import enum
import math
from dataclasses import dataclass, field
from typing import Optional, Sequence

from . import _lib as L


class MultiStreamError(RuntimeError):
    """reduction.hpp:91"""


class PlanError(RuntimeError):
    """mapping.hpp:209"""


class PipelineError(RuntimeError):
    """channels.hpp:105"""


class ConfigError(RuntimeError):
    """config.hpp:39"""


L.register_error(L.GMI_ERR_INVALID, ValueError)
L.register_error(L.GMI_ERR_MULTISTREAM, MultiStreamError)
L.register_error(L.GMI_ERR_PLAN, PlanError)
L.register_error(L.GMI_ERR_PIPELINE, PipelineError)
L.register_error(L.GMI_ERR_CONFIG, ConfigError)
L.register_error(L.GMI_ERR_DOMAIN, RuntimeError)


def _lib():
    return L.lib()


def _ints(values) -> C.Array:
    values = list(values)
    return (C.c_int * max(1, len(values)))(*values)


# ------------------------------------------------------------------ reduction.hpp
class Strategy(enum.IntEnum):
    MPR = 0
    MRR = 1
    HAR = 2


class LinkKind(enum.IntEnum):
    Intra = 0
    HostBounce = 1
    Ring = 2
    LocalReduce = 3


LINK_NAMES = {LinkKind.Intra: "intra", LinkKind.HostBounce: "host_bounce", LinkKind.Ring: "ring",
              LinkKind.LocalReduce: "local_reduce"}


def to_string(x) -> str:
    if isinstance(x, Strategy):
        return x.name
    if isinstance(x, LinkKind):
        return LINK_NAMES[x]
    if isinstance(x, TemplateKind):
        return "async_decoupled" if x == TemplateKind.AsyncDecoupled else x.name
    if isinstance(x, Role):
        return x.name.lower()
    raise TypeError(type(x))


@dataclass
class GmiLayout:
    mpl: list = field(default_factory=list)

    def num_gpus(self) -> int:
        return len(self.mpl)

    def total_gmis(self) -> int:
        return sum(len(l) for l in self.mpl)

    def uniform(self) -> bool:
        return all(len(l) == len(self.mpl[0]) for l in self.mpl)

    def all_gmis(self) -> list:
        return [i for l in self.mpl for i in l]

    def validate(self) -> None:
        # same checks as select_strategy's first step; raised from libgmi
        counts, ids = self._flat()
        out = C.c_int()
        L.check(_lib().gmi_select_strategy(len(self.mpl), counts, ids, C.byref(out)))

    def _flat(self):
        return _ints(len(l) for l in self.mpl), _ints(self.all_gmis())


def _layout(x) -> GmiLayout:
    return x if isinstance(x, GmiLayout) else GmiLayout([list(l) for l in x])


@dataclass
class GradientBuffer:
    gmi_id: int
    values: Sequence[float]


@dataclass
class TraceEvent:
    step: int
    src: int
    dst: int
    bytes: float
    kind: LinkKind


@dataclass
class ReductionRun:
    strategy: Strategy = Strategy.MPR
    result: list = field(default_factory=list)
    latency: float = 0.0
    broadcast_latency: float = 0.0
    trace: list = field(default_factory=list)


def select_strategy(layout) -> Strategy:
    lay = _layout(layout)
    counts, ids = lay._flat()
    out = C.c_int()
    L.check(_lib().gmi_select_strategy(len(lay.mpl), counts, ids, C.byref(out)))
    return Strategy(out.value)


def leader_gmis(layout) -> list:
    lay = _layout(layout)
    counts, ids = lay._flat()
    out = (C.c_int * max(1, len(lay.mpl)))()
    L.check(_lib().gmi_leader_gmis(len(lay.mpl), counts, ids, out))
    return list(out[: len(lay.mpl)])


def mrr_rings(layout) -> list:
    lay = _layout(layout)
    counts, ids = lay._flat()
    out = (C.c_int * max(1, lay.total_gmis()))()
    t = C.c_int()
    L.check(_lib().gmi_mrr_rings(len(lay.mpl), counts, ids, out, C.byref(t)))
    g = len(lay.mpl)
    return [list(out[r * g:(r + 1) * g]) for r in range(t.value)]


def predict_latency(s, g: int, t: int, m_p: float, b1: float, b2: float) -> float:
    out = C.c_double()
    L.check(_lib().gmi_predict_latency(int(s), g, t, float(m_p), float(b1), float(b2), C.byref(out)))
    return out.value


def reduction_schedule(strategy, layout, length: int, b1: float, b2: float, elem_bytes: float = 8.0):
    """Trace + latencies of execute() without touching element data."""
    lay = _layout(layout)
    counts, ids = lay._flat()
    info = L.ReductionInfo()
    L.check(_lib().gmi_reduction_schedule(int(strategy), len(lay.mpl), counts, ids, length,
                                          elem_bytes, b1, b2, None, 0, C.byref(info)))
    trace = (L.TraceEvent * max(1, info.trace_len))()
    L.check(_lib().gmi_reduction_schedule(int(strategy), len(lay.mpl), counts, ids, length,
                                          elem_bytes, b1, b2, trace, info.trace_len, C.byref(info)))
    events = [TraceEvent(e.step, e.src, e.dst, e.bytes, LinkKind(e.kind))
              for e in trace[: info.trace_len]]
    return info, events


def _check_buffers(layout: GmiLayout, buffers) -> int:
    layout.validate()
    members = layout.all_gmis()
    if len(buffers) != len(members):
        raise ValueError("need exactly one buffer per GMI in the layout")
    length = len(buffers[0].values) if buffers else 0
    seen = set()
    for b in buffers:
        if len(b.values) != length:
            raise ValueError("mismatched buffer lengths")
        if b.gmi_id in seen:
            raise ValueError(f"duplicate buffer for gmi {b.gmi_id}")
        seen.add(b.gmi_id)
    for i in members:
        if i not in seen:
            raise ValueError(f"missing buffer for gmi {i}")
    return length


def execute(strategy, layout, buffers, topo: "Topology", device="cuda"):
    """Device-backed execute() (reduction.hpp:225-334): fp64 buffers are copied to the GPU,
    reduced by the K1 kernel in the reference's fold order, and copied back."""
    import torch

    lay = _layout(layout)
    length = _check_buffers(lay, buffers)
    strategy = Strategy(int(strategy))
    info, trace = reduction_schedule(strategy, lay, length, topo.b1, topo.b2)  # raises MRR errors
    by_id = {b.gmi_id: b for b in buffers}
    dev = [torch.as_tensor(list(by_id[i].values), dtype=torch.float64).to(device)
           for i in lay.all_gmis()]
    out = torch.empty(length, dtype=torch.float64, device=device)
    ptrs = (C.c_void_p * max(1, len(dev)))(*[t.data_ptr() for t in dev])
    counts, ids = lay._flat()
    stream = torch.cuda.current_stream().cuda_stream
    L.check(_lib().gmi_reduce_device(int(strategy), len(lay.mpl), counts, ids, ptrs,
                                     C.c_void_p(out.data_ptr()), length, 1, 0, C.c_void_p(stream)))
    result = out.cpu().tolist()
    return ReductionRun(strategy, result, info.latency, info.broadcast_latency, trace)


# ------------------------------------------------------------------ topology.hpp
class GpuArch(enum.IntEnum):
    SM70 = 70
    SM80 = 80
    SM100 = 100  # B200 extension


class Backend(enum.IntEnum):
    MPS = 0
    MIG = 1


class TaskMode(enum.IntEnum):
    Training = 0
    Serving = 1


MIG_PROFILES = {"1g.5gb": (1, 5.0), "2g.10gb": (2, 10.0), "3g.20gb": (3, 20.0),
                "4g.20gb": (4, 20.0), "7g.40gb": (7, 40.0)}
# B200 (sm100, 180 GB) profiles as NVIDIA publishes them (compute slices of 7, label memory):
# host/catalog.cpp mig_table_sm100; validate_layout also checks the 8 memory slices.
MIG_PROFILES.update({"1g.23gb": (1, 23.0), "1g.45gb": (1, 45.0), "2g.45gb": (2, 45.0), "3g.90gb": (3, 90.0),
                     "4g.90gb": (4, 90.0), "7g.180gb": (7, 180.0)})


@dataclass
class GpuSpec:
    id: int = 0
    arch: GpuArch = GpuArch.SM80
    sm_units: int = 8
    mem_gb: float = 40.0


@dataclass
class GmiPartition:
    gmi_id: int = 0
    gpu_id: int = 0
    backend: Backend = Backend.MPS
    sm_share: float = 1.0
    mem_gb: float = 0.0


def mig_partition(gmi_id: int, gpu_id: int, profile: str) -> GmiPartition:
    if profile not in MIG_PROFILES:
        raise ValueError("unknown MIG profile: " + profile)
    units, mem = MIG_PROFILES[profile]
    return GmiPartition(gmi_id, gpu_id, Backend.MIG, units / 8.0, mem)


def mps_partition(gmi_id: int, gpu_id: int, sm_share: float, mem_gb: float) -> GmiPartition:
    return GmiPartition(gmi_id, gpu_id, Backend.MPS, sm_share, mem_gb)


@dataclass
class Topology:
    gpus: list = field(default_factory=list)
    partitions: list = field(default_factory=list)
    b1: float = 1.0
    b2: float = 30.0

    def _c(self):
        g = (L.GpuT * max(1, len(self.gpus)))(*[L.GpuT(x.id, int(x.arch), x.sm_units, x.mem_gb) for x in self.gpus])
        p = (L.PartitionT * max(1, len(self.partitions)))(
            *[L.PartitionT(x.gmi_id, x.gpu_id, int(x.backend), x.sm_share, x.mem_gb) for x in self.partitions])
        t = L.TopologyT(g, len(self.gpus), p, len(self.partitions), self.b1, self.b2)
        t._keep = (g, p)
        return t


def green_sms(share: float, sm_units: int = 8) -> int:
    """B200 extension: SMs of the green context realising an MPS `share` on an sm100 GPU
    (whole 8-SM groups of 148 SMs, or of sm_units when > 8)."""
    n = C.c_int()
    L.check(_lib().gmi_green_sms(float(share), int(sm_units), C.byref(n)))
    return n.value


def default_topology(num_gpus: int = 2) -> Topology:
    return Topology([GpuSpec(i) for i in range(num_gpus)])


@dataclass
class Violation:
    gpu_id: int
    rule: str


def validate_layout(topo: Topology) -> list:
    t = topo._c()
    n = C.c_int()
    cap = 4 * (len(topo.partitions) + len(topo.gpus)) + 4
    out = (L.ViolationT * cap)()
    L.check(_lib().gmi_validate_layout(C.byref(t), out, cap, C.byref(n)))
    return [Violation(v.gpu_id, v.rule.decode()) for v in out[: n.value]]


def select_backend(arch, mode) -> Backend:
    out = C.c_int()
    L.check(_lib().gmi_select_backend(int(arch), 1 if mode == TaskMode.Training else 0, C.byref(out)))
    return Backend(out.value)


def path_bandwidth(topo: Topology, src: int, dst: int):
    t = topo._c()
    kind, bw = C.c_int(), C.c_double()
    L.check(_lib().gmi_path_bandwidth(C.byref(t), src, dst, C.byref(kind), C.byref(bw)))
    return LinkKind(kind.value), bw.value


# ------------------------------------------------------------------ workload.hpp
class Role(enum.IntEnum):
    Simulator = 1
    Agent = 2
    Trainer = 4


@dataclass
class RoleProfile:
    role: Role
    r_sm: float
    r_mem: float
    t_iter: float


@dataclass
class DrlWorkload:
    name: str = ""
    state_bytes: float = 0.0
    action_bytes: float = 0.0
    reward_bytes: float = 0.0
    model_bytes: float = 0.0
    steps_per_train: int = 1
    alpha: float = 0.2
    beta: float = 0.3
    policy_dims: list = field(default_factory=list)
    simulator: RoleProfile = field(default_factory=lambda: RoleProfile(Role.Simulator, 1.0, 0.5, 6.0))
    agent: RoleProfile = field(default_factory=lambda: RoleProfile(Role.Agent, 0.1, 0.05, 1.0))
    trainer: RoleProfile = field(default_factory=lambda: RoleProfile(Role.Trainer, 0.2, 0.1, 2.0))

    def record_bytes(self) -> float:
        return self.state_bytes + self.action_bytes + self.reward_bytes

    def interaction_time(self) -> float:
        return self.simulator.t_iter + self.agent.t_iter

    def iteration_time(self) -> float:
        return self.interaction_time() + self.trainer.t_iter

    def _c(self) -> L.WorkloadT:
        w = L.WorkloadT()
        w.name = self.name.encode()[:31]
        w.state_bytes, w.action_bytes = self.state_bytes, self.action_bytes
        w.reward_bytes, w.model_bytes = self.reward_bytes, self.model_bytes
        w.steps_per_train, w.alpha, w.beta = self.steps_per_train, self.alpha, self.beta
        if len(self.policy_dims) > L.MAX_DIMS:
            raise ValueError("too many policy dims")
        w.num_dims = len(self.policy_dims)
        for i, d in enumerate(self.policy_dims):
            w.policy_dims[i] = d
        for dst, src in ((w.simulator, self.simulator), (w.agent, self.agent), (w.trainer, self.trainer)):
            dst.r_sm, dst.r_mem, dst.t_iter = src.r_sm, src.r_mem, src.t_iter
        return w

    @staticmethod
    def _from_c(w: L.WorkloadT) -> "DrlWorkload":
        return DrlWorkload(
            w.name.decode(), w.state_bytes, w.action_bytes, w.reward_bytes, w.model_bytes,
            w.steps_per_train, w.alpha, w.beta, list(w.policy_dims[: w.num_dims]),
            RoleProfile(Role.Simulator, w.simulator.r_sm, w.simulator.r_mem, w.simulator.t_iter),
            RoleProfile(Role.Agent, w.agent.r_sm, w.agent.r_mem, w.agent.t_iter),
            RoleProfile(Role.Trainer, w.trainer.r_sm, w.trainer.r_mem, w.trainer.t_iter))


def benchmark_names() -> list:
    return ["AT", "AY", "BB", "FC", "HM", "SH"]


def load_benchmark(name: str) -> DrlWorkload:
    w = L.WorkloadT()
    L.check(_lib().gmi_load_benchmark(name.encode(), C.byref(w)))
    return DrlWorkload._from_c(w)


def validate_workload(w: DrlWorkload) -> None:
    c = w._c()
    L.check(_lib().gmi_validate_workload(C.byref(c)))


def dense_param_count(dims) -> int:
    out = C.c_size_t()
    L.check(_lib().gmi_dense_param_count(_ints(dims), len(dims), C.byref(out)))
    return out.value


def policy_value_param_count(dims) -> int:
    out = C.c_size_t()
    L.check(_lib().gmi_policy_value_param_count(_ints(dims), len(dims), C.byref(out)))
    return out.value


# ------------------------------------------------------------------ mapping.hpp
class TemplateKind(enum.IntEnum):
    TDG = 0
    TCG = 1
    TDG_EX = 2
    TCG_EX = 3
    AsyncDecoupled = 4


class RunMode(enum.IntEnum):
    Serving = 0
    SyncTrain = 1
    AsyncTrain = 2


def select_template(mode) -> TemplateKind:
    return {RunMode.Serving: TemplateKind.TCG, RunMode.SyncTrain: TemplateKind.TCG_EX,
            RunMode.AsyncTrain: TemplateKind.AsyncDecoupled}[RunMode(mode)]


@dataclass
class CostEstimate:
    resource_size: float = 0.0
    comm_bytes: float = 0.0
    throughput: float = 0.0


def serving_cost(tpl, w: DrlWorkload) -> CostEstimate:
    r, c = C.c_double(), C.c_double()
    wc = w._c()
    L.check(_lib().gmi_serving_cost(int(tpl), C.byref(wc), C.byref(r), C.byref(c)))
    return CostEstimate(r.value, c.value)


def training_cost(tpl, w: DrlWorkload, n_gmis: int) -> CostEstimate:
    r, c = C.c_double(), C.c_double()
    wc = w._c()
    L.check(_lib().gmi_training_cost(int(tpl), C.byref(wc), n_gmis, C.byref(r), C.byref(c)))
    return CostEstimate(r.value, c.value)


def allreduce_bytes(n_gmis: int, model_bytes: float) -> float:
    out = C.c_double()
    L.check(_lib().gmi_allreduce_bytes(n_gmis, model_bytes, C.byref(out)))
    return out.value


def _throughput(training, cost, w, r_all, bw):
    out = C.c_double()
    wc = w._c()
    L.check(_lib().gmi_throughput(training, cost.resource_size, cost.comm_bytes, C.byref(wc), r_all, bw,
                                  C.byref(out)))
    return out.value


def serving_throughput(cost, w, r_all, bandwidth):
    return _throughput(0, cost, w, r_all, bandwidth)


def training_throughput(cost, w, r_all, bandwidth):
    return _throughput(1, cost, w, r_all, bandwidth)


@dataclass
class CalibrationParams:
    serving_combw_factor: float = 2.0
    training_combw_factor: float = 7.0


def serving_throughput_ratio(w, cal: CalibrationParams = CalibrationParams()):
    out = C.c_double()
    wc = w._c()
    L.check(_lib().gmi_throughput_ratio(0, C.byref(wc), cal.serving_combw_factor, C.byref(out)))
    return out.value


def training_throughput_ratio(w, cal: CalibrationParams = CalibrationParams()):
    out = C.c_double()
    wc = w._c()
    L.check(_lib().gmi_throughput_ratio(1, C.byref(wc), cal.training_combw_factor, C.byref(out)))
    return out.value


def serving_colocation_penalty(w):
    out = C.c_double()
    wc = w._c()
    L.check(_lib().gmi_colocation_penalty(0, C.byref(wc), C.byref(out)))
    return out.value


def training_colocation_penalty(w):
    out = C.c_double()
    wc = w._c()
    L.check(_lib().gmi_colocation_penalty(1, C.byref(wc), C.byref(out)))
    return out.value


@dataclass
class MappingPlan:
    template_kind: TemplateKind = TemplateKind.TCG
    gmi_assignments: dict = field(default_factory=dict)  # gmi -> set[Role]
    gpu_layout: dict = field(default_factory=dict)       # gpu -> [gmi ids]
    serving_gpus: list = field(default_factory=list)
    training_gpus: list = field(default_factory=list)

    def mpl(self) -> list:
        return [self.gpu_layout[g] for g in sorted(self.gpu_layout)]

    def gmis_with_role(self, r: Role) -> list:
        return [g for g in sorted(self.gmi_assignments) if r in self.gmi_assignments[g]]

    def _c(self):
        gpus = sorted(self.gpu_layout)
        ids = [i for g in gpus for i in self.gpu_layout[g]]
        masks = [sum(int(r) for r in self.gmi_assignments.get(i, ())) for i in ids]
        arrs = (_ints(gpus), _ints(len(self.gpu_layout[g]) for g in gpus), _ints(ids), _ints(masks))
        p = L.PlanT(int(self.template_kind), len(gpus), *arrs)
        p._keep = arrs
        return p


def _roles(mask: int) -> set:
    return {r for r in Role if mask & int(r)}


def build_plan(tpl, topo: Topology, w: DrlWorkload, gmis_per_gpu: int) -> MappingPlan:
    t = topo._c()
    ng = max(1, len(topo.gpus))
    total = max(1, len(topo.gpus) * max(0, gmis_per_gpu))
    gpu_ids, gmi_ids, roles, serving = (C.c_int * ng)(), (C.c_int * total)(), (C.c_int * total)(), (C.c_int * ng)()
    L.check(_lib().gmi_build_plan(int(tpl), C.byref(t), gmis_per_gpu, gpu_ids, gmi_ids, roles, serving))
    plan = MappingPlan(TemplateKind(int(tpl)))
    k = 0
    for gi in range(len(topo.gpus)):
        gpu = gpu_ids[gi]
        plan.gpu_layout[gpu] = list(gmi_ids[k:k + gmis_per_gpu])
        for i in plan.gpu_layout[gpu]:
            plan.gmi_assignments[i] = _roles(roles[i])
        k += gmis_per_gpu
        if serving[gi] == 1:
            plan.serving_gpus.append(gpu)
        elif serving[gi] == 0:
            plan.training_gpus.append(gpu)
    return plan


# ------------------------------------------------------------------ search.hpp
@dataclass
class ProfileResult:
    runnable: bool = False
    top: float = 0.0
    mem: float = 0.0


class Profiler:
    """search.hpp:32-37 — subclass and override profile()."""

    def profile(self, bench: str, gmis_per_gpu: int, num_env: int) -> ProfileResult:
        raise NotImplementedError


@dataclass
class SearchConfig:
    num_env_grid: list = field(default_factory=lambda: [128, 256, 512, 1024, 2048, 4096, 8192, 16384])
    max_gmis_per_gpu: int = 10
    sat_threshold: float = 0.1

    def _c(self):
        g = _ints(self.num_env_grid)
        c = L.SearchConfigT(g, len(self.num_env_grid), self.max_gmis_per_gpu, self.sat_threshold)
        c._keep = g
        return c


def saturation(top, pre_top, mem, pre_mem) -> float:
    out = C.c_double()
    L.check(_lib().gmi_saturation(top, pre_top, mem, pre_mem, C.byref(out)))
    return out.value


@dataclass
class ThroughputEstimator:
    workload: DrlWorkload
    b1: float = 1.0
    b2: float = 30.0
    latency_scale: float = 1000.0

    def _c(self):
        return L.EstimatorT(self.workload._c(), self.b1, self.b2, self.latency_scale)

    def comm_discount(self, gmis_per_gpu: int, num_gpu: int) -> float:
        out = C.c_double()
        e = self._c()
        L.check(_lib().gmi_comm_discount(C.byref(e), gmis_per_gpu, num_gpu, C.byref(out)))
        return out.value

    def estimate(self, gmis_per_gpu: int, num_gpu: int, per_gmi_top: float) -> float:
        out = C.c_double()
        e = self._c()
        L.check(_lib().gmi_estimate(C.byref(e), gmis_per_gpu, num_gpu, per_gmi_top, C.byref(out)))
        return out.value


@dataclass
class SyntheticCostModel(Profiler):
    peak_top: float = 120000.0
    mem_base: float = 1.0
    mem_per_env: float = 0.002
    mem_capacity: float = 40.0
    min_runnable_share: float = 0.1
    knee_base: int = 8192
    knee_override: dict = field(default_factory=dict)
    cap_scale: dict = field(default_factory=dict)

    def _c(self):
        kk, kv = _ints(self.knee_override.keys()), _ints(self.knee_override.values())
        ck = _ints(self.cap_scale.keys())
        cv = (C.c_double * max(1, len(self.cap_scale)))(*self.cap_scale.values())
        m = L.SyntheticModelT(self.peak_top, self.mem_base, self.mem_per_env, self.mem_capacity,
                              self.min_runnable_share, self.knee_base, len(self.knee_override), kk, kv,
                              len(self.cap_scale), ck, cv)
        m._keep = (kk, kv, ck, cv)
        return m

    def profile(self, bench, gmis_per_gpu, num_env):
        m = self._c()
        ok, top, mem = C.c_int(), C.c_double(), C.c_double()
        L.check(_lib().gmi_synthetic_profile(C.byref(m), bench.encode(), gmis_per_gpu, num_env,
                                             C.byref(ok), C.byref(top), C.byref(mem)))
        return ProfileResult(bool(ok.value), top.value, mem.value)


class RecordedTraceProfiler(Profiler):
    def __init__(self, handle):
        self._h = handle

    @staticmethod
    def from_file(path: str) -> "RecordedTraceProfiler":
        h = C.c_void_p()
        L.check(_lib().gmi_trace_profiler_load(path.encode(), C.byref(h)))
        return RecordedTraceProfiler(h)

    def profile(self, bench, gmis_per_gpu, num_env):
        ok, top, mem = C.c_int(), C.c_double(), C.c_double()
        L.check(_lib().gmi_trace_profiler_profile(self._h, bench.encode(), gmis_per_gpu, num_env,
                                                  C.byref(ok), C.byref(top), C.byref(mem)))
        return ProfileResult(bool(ok.value), top.value, mem.value)

    def __del__(self):
        if getattr(self, "_h", None) and L is not None:
            L.lib().gmi_trace_profiler_free(self._h)
            self._h = None


@dataclass
class GpuProfiler(Profiler):
    """B200 measured profiler: runs the real PPO iteration of the benchmark's catalog MLP
    with `gmis_per_gpu` GMIs x `num_env` envs on `device` (gmi_gpu_profile) and reports
    per-GMI env-steps/s and per-GMI device GB -- the on-device Profiler::profile the
    reference leaves to a synthetic model (search.hpp:32-37, 100-132)."""
    device: int = 0
    backend: int = 1  # 1 = SM-partitioned green contexts, 0 = streams
    iters: int = 3

    def profile(self, bench, gmis_per_gpu, num_env):
        ok, top, mem = C.c_int(), C.c_double(), C.c_double()
        L.check(_lib().gmi_gpu_profile(bench.encode(), gmis_per_gpu, num_env, self.device, self.backend,
                                       self.iters, C.byref(ok), C.byref(top), C.byref(mem)))
        return ProfileResult(bool(ok.value), top.value, mem.value)


@dataclass
class VisitedPoint:
    gmis_per_gpu: int
    num_env: int
    runnable: bool
    top: float
    mem: float
    sat: Optional[float]
    acc_top: Optional[float]
    pruned_here: bool


@dataclass
class SearchResult:
    feasible: bool = False
    reason: str = ""
    num_env: int = 0
    gmis_per_gpu: int = 0
    est_throughput: float = 0.0
    visited: list = field(default_factory=list)


def explore(profiler: Profiler, estimator: ThroughputEstimator, bench: str, num_gpu: int,
            config: SearchConfig = None) -> SearchResult:
    config = config or SearchConfig()
    errors = []

    def probe(_user, b, gpg, env, ok, top, mem):
        try:
            r = profiler.profile(b.decode(), gpg, env)
        except BaseException as exc:  # surfaced after the C call returns
            errors.append(exc)
            return L.GMI_ERR_DOMAIN
        ok[0], top[0], mem[0] = int(bool(r.runnable)), float(r.top), float(r.mem)
        return 0

    cb = L.PROBE_FN(probe)
    est = estimator._c()
    cfg = config._c()
    res = L.SearchResultT()
    cap = max(1, config.max_gmis_per_gpu * len(config.num_env_grid))
    visits = (L.VisitT * cap)()
    rc = _lib().gmi_explore(cb, None, C.byref(est), bench.encode(), num_gpu, C.byref(cfg),
                            C.byref(res), visits, cap)
    if errors:
        raise errors[0]
    L.check(rc)
    out = SearchResult(bool(res.feasible), res.reason.decode(), res.num_env, res.gmis_per_gpu,
                       res.est_throughput)
    for v in visits[: res.num_visited]:
        out.visited.append(VisitedPoint(v.gmis_per_gpu, v.num_env, bool(v.runnable), v.top, v.mem,
                                        v.sat if v.has_sat else None,
                                        v.acc_top if v.has_acc_top else None, bool(v.pruned_here)))
    return out


# ------------------------------------------------------------------ channels.hpp
class BatchMode(enum.IntEnum):
    Slice = 0
    Stack = 1


@dataclass
class PipelineConfig:
    compress_threshold: int = 8
    batch_mode: BatchMode = BatchMode.Stack
    target_batch: int = 32
    per_message_overhead: float = 1.0
    seed: int = 0

    def _c(self):
        return L.PipelineConfigT(self.compress_threshold, int(self.batch_mode), self.target_batch,
                                 self.per_message_overhead, self.seed)


def uni_channel(config: PipelineConfig) -> PipelineConfig:
    from dataclasses import replace
    return replace(config, compress_threshold=1)


@dataclass
class RecordId:
    agent_gmi: int
    seq: int


@dataclass
class TrainingBatch:
    trainer_gmi: int
    emit_time: float
    records: list


@dataclass
class PipelineMetrics:
    pps: float = 0.0
    ttop: float = 0.0
    records_produced: int = 0
    records_delivered: int = 0
    units_sent: int = 0
    batches_emitted: int = 0
    bytes_moved: float = 0.0
    transfer_busy_time: float = 0.0
    delivery_makespan: float = 0.0
    training_makespan: float = 0.0
    trainer_records: dict = field(default_factory=dict)
    batches: list = field(default_factory=list)


def simulate_pipeline(w: DrlWorkload, plan: MappingPlan, topo: Topology, config: PipelineConfig,
                      duration: float) -> PipelineMetrics:
    wc, pc, tc, cc = w._c(), plan._c(), topo._c(), config._c()
    h = C.c_void_p()
    m = L.PipelineMetricsT()
    L.check(_lib().gmi_simulate_pipeline(C.byref(wc), C.byref(pc), C.byref(tc), C.byref(cc),
                                         float(duration), C.byref(h), C.byref(m)))
    return _metrics_from_handle(h, m)


def run_channels_device(w: DrlWorkload, plan: MappingPlan, topo: Topology, config: PipelineConfig,
                        duration: float, agent_bufs: list, trainer_bufs: list, trainer_capacity: int,
                        stream: int = 0) -> PipelineMetrics:
    """The channel pipeline on the GPU (gmi_channel_run): agent_bufs = device pointers
    [channel * agents + agent] (state / action / reward, agents in ascending gmi id),
    trainer_bufs likewise per trainer (receive buffers of trainer_capacity records)."""
    wc, pc, tc, cc = w._c(), plan._c(), topo._c(), config._c()
    h = C.c_void_p()
    m = L.PipelineMetricsT()
    ab = (C.c_void_p * len(agent_bufs))(*agent_bufs)
    tb = (C.c_void_p * len(trainer_bufs))(*trainer_bufs)
    L.check(_lib().gmi_channel_run(C.byref(wc), C.byref(pc), C.byref(tc), C.byref(cc), float(duration), ab,
                                   len(agent_bufs), tb, len(trainer_bufs), int(trainer_capacity),
                                   C.c_void_p(stream), C.byref(h), C.byref(m)))
    return _metrics_from_handle(h, m)


def _metrics_from_handle(h, m) -> PipelineMetrics:
    try:
        out = PipelineMetrics(m.pps, m.ttop, m.records_produced, m.records_delivered, m.units_sent,
                              m.batches_emitted, m.bytes_moved, m.transfer_busy_time,
                              m.delivery_makespan, m.training_makespan)
        n = m.num_trainers
        tr, rec = (C.c_int * max(1, n))(), (C.c_long * max(1, n))()
        L.check(_lib().gmi_pipeline_trainer_records(h, tr, rec))
        out.trainer_records = {tr[i]: rec[i] for i in range(n)}
        for i in range(_lib().gmi_pipeline_num_batches(h)):
            t, e, k = C.c_int(), C.c_double(), C.c_size_t()
            L.check(_lib().gmi_pipeline_batch(h, i, C.byref(t), C.byref(e), C.byref(k)))
            ag, sq = (C.c_int * max(1, k.value))(), (C.c_long * max(1, k.value))()
            L.check(_lib().gmi_pipeline_batch_records(h, i, ag, sq))
            out.batches.append(TrainingBatch(t.value, e.value,
                                             [RecordId(ag[j], sq[j]) for j in range(k.value)]))
        return out
    finally:
        _lib().gmi_pipeline_free(h)


# ------------------------------------------------------------------ config.hpp
@dataclass
class ModelParams:
    calibration: CalibrationParams = field(default_factory=CalibrationParams)
    gmis_per_gpu: int = 2
    latency_scale: float = 1000.0
    pipeline: PipelineConfig = field(default_factory=PipelineConfig)


@dataclass
class SearchSettings:
    config: SearchConfig = field(default_factory=SearchConfig)
    profile_trace: Optional[str] = None


class ConfigFile:
    def __init__(self, handle):
        self._h = handle

    def __del__(self):
        if getattr(self, "_h", None) and L is not None:
            L.lib().gmi_config_free(self._h)
            self._h = None

    def has(self, section: str) -> bool:
        out = C.c_int()
        L.check(_lib().gmi_config_has(self._h, section.encode(), C.byref(out)))
        return bool(out.value)

    def get(self, section: str, key: str) -> Optional[str]:
        buf = C.create_string_buffer(4096)
        found = C.c_int()
        L.check(_lib().gmi_config_get(self._h, section.encode(), key.encode(), buf, 4096, C.byref(found)))
        return buf.value.decode() if found.value else None


def parse_config(text: str, origin: str = "<config>") -> ConfigFile:
    h = C.c_void_p()
    L.check(_lib().gmi_config_parse(text.encode(), origin.encode(), C.byref(h)))
    return ConfigFile(h)


def load_config(path: str) -> ConfigFile:
    h = C.c_void_p()
    L.check(_lib().gmi_config_load(path.encode(), C.byref(h)))
    return ConfigFile(h)


def topology_from_config(cfg: ConfigFile) -> Topology:
    ng, np_, b1, b2 = C.c_int(), C.c_int(), C.c_double(), C.c_double()
    L.check(_lib().gmi_config_topology(cfg._h, None, 0, C.byref(ng), None, 0, C.byref(np_), C.byref(b1), C.byref(b2)))
    g, p = (L.GpuT * max(1, ng.value))(), (L.PartitionT * max(1, np_.value))()
    L.check(_lib().gmi_config_topology(cfg._h, g, ng.value, C.byref(ng), p, np_.value, C.byref(np_),
                                       C.byref(b1), C.byref(b2)))
    return Topology([GpuSpec(x.id, GpuArch(x.arch), x.sm_units, x.mem_gb) for x in g[: ng.value]],
                    [GmiPartition(x.gmi_id, x.gpu_id, Backend(x.backend), x.sm_share, x.mem_gb)
                     for x in p[: np_.value]], b1.value, b2.value)


def workload_from_config(cfg: ConfigFile, fallback: str = "AT") -> DrlWorkload:
    w = L.WorkloadT()
    L.check(_lib().gmi_config_workload(cfg._h, fallback.encode(), C.byref(w)))
    return DrlWorkload._from_c(w)


def model_from_config(cfg: ConfigFile) -> ModelParams:
    m = L.ModelParamsT()
    L.check(_lib().gmi_config_model(cfg._h, C.byref(m)))
    p = m.pipeline
    return ModelParams(CalibrationParams(m.serving_combw_factor, m.training_combw_factor), m.gmis_per_gpu,
                       m.latency_scale, PipelineConfig(p.compress_threshold, BatchMode(p.batch_mode),
                                                       p.target_batch, p.per_message_overhead, p.seed))


def search_from_config(cfg: ConfigFile) -> SearchSettings:
    s = L.SearchSettingsT()
    L.check(_lib().gmi_config_search(cfg._h, C.byref(s)))
    return SearchSettings(SearchConfig(list(s.grid[: s.grid_len]), s.max_gmis_per_gpu, s.sat_threshold),
                          s.profile_trace.decode() if s.has_profile_trace else None)
