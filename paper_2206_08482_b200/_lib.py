"""ctypes binding of libgmi.so (C-ABI declared in include/gmi.h).

The library is built in-tree by ``__graft_entry__.build()``.  There is no
Python or CPU fallback: a missing library raises immediately.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libgmi.so")

_lib = None

c_int_p = C.POINTER(C.c_int)
c_double_p = C.POINTER(C.c_double)
c_float_p = C.POINTER(C.c_float)

# ------------------------------------------------------------------ C structs (gmi.h)
MAX_DIMS = 16
MAX_GRID = 32


class TraceEvent(C.Structure):
    _fields_ = [("step", C.c_int), ("src", C.c_int), ("dst", C.c_int), ("kind", C.c_int),
                ("bytes", C.c_double)]


class ReductionInfo(C.Structure):
    _fields_ = [("strategy", C.c_int), ("result_holder", C.c_int), ("latency", C.c_double),
                ("broadcast_latency", C.c_double), ("trace_len", C.c_size_t)]


class GpuT(C.Structure):
    _fields_ = [("id", C.c_int), ("arch", C.c_int), ("sm_units", C.c_int), ("mem_gb", C.c_double)]


class PartitionT(C.Structure):
    _fields_ = [("gmi_id", C.c_int), ("gpu_id", C.c_int), ("backend", C.c_int),
                ("sm_share", C.c_double), ("mem_gb", C.c_double)]


class TopologyT(C.Structure):
    _fields_ = [("gpus", C.POINTER(GpuT)), ("num_gpus", C.c_int), ("parts", C.POINTER(PartitionT)),
                ("num_parts", C.c_int), ("b1", C.c_double), ("b2", C.c_double)]


class ViolationT(C.Structure):
    _fields_ = [("gpu_id", C.c_int), ("rule", C.c_char * 160)]


class RoleProfileT(C.Structure):
    _fields_ = [("r_sm", C.c_double), ("r_mem", C.c_double), ("t_iter", C.c_double)]


class WorkloadT(C.Structure):
    _fields_ = [("name", C.c_char * 32), ("state_bytes", C.c_double), ("action_bytes", C.c_double),
                ("reward_bytes", C.c_double), ("model_bytes", C.c_double),
                ("steps_per_train", C.c_int), ("alpha", C.c_double), ("beta", C.c_double),
                ("num_dims", C.c_int), ("policy_dims", C.c_int * MAX_DIMS),
                ("simulator", RoleProfileT), ("agent", RoleProfileT), ("trainer", RoleProfileT)]


PROBE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_char_p, C.c_int, C.c_int, c_int_p, c_double_p,
                       c_double_p)


class SearchConfigT(C.Structure):
    _fields_ = [("num_env_grid", c_int_p), ("grid_len", C.c_int), ("max_gmis_per_gpu", C.c_int),
                ("sat_threshold", C.c_double)]


class EstimatorT(C.Structure):
    _fields_ = [("workload", WorkloadT), ("b1", C.c_double), ("b2", C.c_double),
                ("latency_scale", C.c_double)]


class VisitT(C.Structure):
    _fields_ = [("gmis_per_gpu", C.c_int), ("num_env", C.c_int), ("runnable", C.c_int),
                ("top", C.c_double), ("mem", C.c_double), ("has_sat", C.c_int), ("sat", C.c_double),
                ("has_acc_top", C.c_int), ("acc_top", C.c_double), ("pruned_here", C.c_int)]


class SearchResultT(C.Structure):
    _fields_ = [("feasible", C.c_int), ("reason", C.c_char * 96), ("num_env", C.c_int),
                ("gmis_per_gpu", C.c_int), ("est_throughput", C.c_double), ("num_visited", C.c_size_t)]


class SyntheticModelT(C.Structure):
    _fields_ = [("peak_top", C.c_double), ("mem_base", C.c_double), ("mem_per_env", C.c_double),
                ("mem_capacity", C.c_double), ("min_runnable_share", C.c_double),
                ("knee_base", C.c_int), ("num_knee", C.c_int), ("knee_keys", c_int_p),
                ("knee_values", c_int_p), ("num_cap", C.c_int), ("cap_keys", c_int_p),
                ("cap_values", c_double_p)]


class PipelineConfigT(C.Structure):
    _fields_ = [("compress_threshold", C.c_int), ("batch_mode", C.c_int), ("target_batch", C.c_int),
                ("per_message_overhead", C.c_double), ("seed", C.c_uint)]


class PipelineMetricsT(C.Structure):
    _fields_ = [("pps", C.c_double), ("ttop", C.c_double), ("records_produced", C.c_long),
                ("records_delivered", C.c_long), ("units_sent", C.c_long),
                ("batches_emitted", C.c_long), ("bytes_moved", C.c_double),
                ("transfer_busy_time", C.c_double), ("delivery_makespan", C.c_double),
                ("training_makespan", C.c_double), ("num_trainers", C.c_size_t)]


class PlanT(C.Structure):
    _fields_ = [("template_kind", C.c_int), ("num_gpus", C.c_int), ("gpu_ids", c_int_p),
                ("counts", c_int_p), ("gmi_ids", c_int_p), ("role_masks", c_int_p)]


class ModelParamsT(C.Structure):
    _fields_ = [("serving_combw_factor", C.c_double), ("training_combw_factor", C.c_double),
                ("gmis_per_gpu", C.c_int), ("latency_scale", C.c_double),
                ("pipeline", PipelineConfigT)]


class SearchSettingsT(C.Structure):
    _fields_ = [("grid", C.c_int * MAX_GRID), ("grid_len", C.c_int), ("max_gmis_per_gpu", C.c_int),
                ("sat_threshold", C.c_double), ("has_profile_trace", C.c_int),
                ("profile_trace", C.c_char * 512)]


P = C.POINTER
vp = C.c_void_p
ci = C.c_int
cd = C.c_double
csz = C.c_size_t
cll = C.c_longlong

# name -> (restype, argtypes); kept in sync with include/gmi.h (tests check both ways).
PROTOTYPES: dict[str, tuple] = {
    "gmi_last_error": (C.c_char_p, []),
    "gmi_exit_code": (ci, [ci]),
    "gmi_version": (ci, []),
    "gmi_select_strategy": (ci, [ci, c_int_p, c_int_p, c_int_p]),
    "gmi_leader_gmis": (ci, [ci, c_int_p, c_int_p, c_int_p]),
    "gmi_mrr_rings": (ci, [ci, c_int_p, c_int_p, c_int_p, c_int_p]),
    "gmi_predict_latency": (ci, [ci, ci, ci, cd, cd, cd, c_double_p]),
    "gmi_reduction_schedule": (ci, [ci, ci, c_int_p, c_int_p, csz, cd, cd, cd, P(TraceEvent), csz,
                                    P(ReductionInfo)]),
    "gmi_reduce_device": (ci, [ci, ci, c_int_p, c_int_p, P(vp), vp, csz, ci, ci, vp]),
    "gmi_allreduce": (ci, [ci, ci, c_int_p, c_int_p, P(vp), csz, ci, P(vp), cd, cd, P(ReductionInfo)]),
    "gmi_validate_layout": (ci, [P(TopologyT), P(ViolationT), ci, c_int_p]),
    "gmi_green_sms": (ci, [C.c_double, ci, c_int_p]),
    "gmi_select_backend": (ci, [ci, ci, c_int_p]),
    "gmi_path_bandwidth": (ci, [P(TopologyT), ci, ci, c_int_p, c_double_p]),
    "gmi_load_benchmark": (ci, [C.c_char_p, P(WorkloadT)]),
    "gmi_validate_workload": (ci, [P(WorkloadT)]),
    "gmi_dense_param_count": (ci, [c_int_p, ci, P(csz)]),
    "gmi_policy_value_param_count": (ci, [c_int_p, ci, P(csz)]),
    "gmi_serving_cost": (ci, [ci, P(WorkloadT), c_double_p, c_double_p]),
    "gmi_training_cost": (ci, [ci, P(WorkloadT), ci, c_double_p, c_double_p]),
    "gmi_allreduce_bytes": (ci, [ci, cd, c_double_p]),
    "gmi_throughput": (ci, [ci, cd, cd, P(WorkloadT), cd, cd, c_double_p]),
    "gmi_throughput_ratio": (ci, [ci, P(WorkloadT), cd, c_double_p]),
    "gmi_colocation_penalty": (ci, [ci, P(WorkloadT), c_double_p]),
    "gmi_build_plan": (ci, [ci, P(TopologyT), ci, c_int_p, c_int_p, c_int_p, c_int_p]),
    "gmi_saturation": (ci, [cd, cd, cd, cd, c_double_p]),
    "gmi_comm_discount": (ci, [P(EstimatorT), ci, ci, c_double_p]),
    "gmi_estimate": (ci, [P(EstimatorT), ci, ci, cd, c_double_p]),
    "gmi_explore": (ci, [PROBE_FN, vp, P(EstimatorT), C.c_char_p, ci, P(SearchConfigT),
                         P(SearchResultT), P(VisitT), csz]),
    "gmi_synthetic_model_defaults": (None, [P(SyntheticModelT)]),
    "gmi_synthetic_profile": (ci, [P(SyntheticModelT), C.c_char_p, ci, ci, c_int_p, c_double_p,
                                   c_double_p]),
    "gmi_trace_profiler_load": (ci, [C.c_char_p, P(vp)]),
    "gmi_trace_profiler_profile": (ci, [vp, C.c_char_p, ci, ci, c_int_p, c_double_p, c_double_p]),
    "gmi_trace_profiler_free": (None, [vp]),
    "gmi_gpu_profile": (ci, [C.c_char_p, ci, ci, ci, ci, ci, c_int_p, c_double_p, c_double_p]),
    "gmi_gpu_probe": (ci, [vp, C.c_char_p, ci, ci, c_int_p, c_double_p, c_double_p]),
    "gmi_pipeline_config_defaults": (None, [P(PipelineConfigT)]),
    "gmi_simulate_pipeline": (ci, [P(WorkloadT), P(PlanT), P(TopologyT), P(PipelineConfigT), cd,
                                   P(vp), P(PipelineMetricsT)]),
    "gmi_channel_run": (ci, [P(WorkloadT), P(PlanT), P(TopologyT), P(PipelineConfigT), cd, P(vp), ci, P(vp), ci,
                             C.c_long, vp, P(vp), P(PipelineMetricsT)]),
    "gmi_pipeline_trainer_records": (ci, [vp, c_int_p, P(C.c_long)]),
    "gmi_pipeline_num_batches": (csz, [vp]),
    "gmi_pipeline_batch": (ci, [vp, csz, c_int_p, c_double_p, P(csz)]),
    "gmi_pipeline_batch_records": (ci, [vp, csz, c_int_p, P(C.c_long)]),
    "gmi_pipeline_free": (None, [vp]),
    "gmi_config_parse": (ci, [C.c_char_p, C.c_char_p, P(vp)]),
    "gmi_config_load": (ci, [C.c_char_p, P(vp)]),
    "gmi_config_has": (ci, [vp, C.c_char_p, c_int_p]),
    "gmi_config_topology": (ci, [vp, P(GpuT), ci, c_int_p, P(PartitionT), ci, c_int_p, c_double_p,
                                 c_double_p]),
    "gmi_config_workload": (ci, [vp, C.c_char_p, P(WorkloadT)]),
    "gmi_config_model": (ci, [vp, P(ModelParamsT)]),
    "gmi_config_search": (ci, [vp, P(SearchSettingsT)]),
    "gmi_config_get": (ci, [vp, C.c_char_p, C.c_char_p, C.c_char_p, csz, c_int_p]),
    "gmi_config_free": (None, [vp]),
    "gmi_dev_gemm": (ci, [ci, ci, ci, ci, ci, ci, vp, cll, vp, cll, vp, cll, vp, vp, cll, ci, ci, vp]),
}

# Error codes (gmi.h)
GMI_OK, GMI_ERR_DOMAIN, GMI_ERR_INVALID, GMI_ERR_MULTISTREAM, GMI_ERR_PLAN = 0, 1, 2, 3, 4
GMI_ERR_PIPELINE, GMI_ERR_CONFIG, GMI_ERR_CUDA, GMI_ERR_NCCL = 5, 6, 7, 8


class GmiError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"libgmi.so not built at {LIB_PATH}; run __graft_entry__.build() "
                "(no CPU fallback exists)")
        handle = C.CDLL(LIB_PATH, mode=C.RTLD_GLOBAL)
        for name, (res, args) in PROTOTYPES.items():
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        _lib = handle
    return _lib


_error_types: dict[int, type] = {}


def register_error(code: int, exc: type) -> None:
    _error_types[code] = exc


def check(code: int) -> None:
    if code != 0:
        msg = lib().gmi_last_error().decode(errors="replace")
        exc = _error_types.get(code)
        if exc is not None:
            raise exc(msg)
        raise GmiError(code, msg)


def call(name: str, *args) -> None:
    check(getattr(lib(), name)(*args))
