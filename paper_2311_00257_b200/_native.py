"""ctypes binding of include/amsp_c.h (libamsp.so).

The library is built in-tree by paper_2311_00257_b200/build.py. Loading is
mandatory: there is no Python or CPU fallback for any entry point, and a
missing library raises immediately.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

PKG = Path(__file__).resolve().parent
LIB_PATH = PKG / "libamsp.so"

AMSP_OK, AMSP_EINVAL, AMSP_EINFEASIBLE, AMSP_ECUDA = 0, 1, 2, 3


class AmspError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


class InvalidConfig(AmspError):
    pass


class Infeasible(AmspError):
    pass


class CudaError(AmspError):
    pass


class Mesh(C.Structure):
    _fields_ = [("per_node", C.c_int), ("nodes", C.c_int)]


class Plan(C.Structure):
    _fields_ = [("p", Mesh), ("g", Mesh), ("os", Mesh), ("has_secondary", C.c_int),
                ("secondary", Mesh)]


class Cluster(C.Structure):
    _fields_ = [("gpus_per_node", C.c_int), ("node_count", C.c_int),
                ("gpu_memory_capacity", C.c_uint64), ("dp_mesh", Mesh),
                ("leaf_count", C.c_int), ("nodes_per_leaf", C.c_int),
                ("inter_leaf_penalty", C.c_double)]


class Model(C.Structure):
    _fields_ = [("total_params", C.c_uint64), ("layer_count", C.c_int),
                ("modules_per_layer", C.c_int), ("module_params", C.POINTER(C.c_uint64)),
                ("hidden", C.c_int), ("seq_len", C.c_int), ("micro_batch", C.c_int),
                ("micro_batch_count", C.c_int), ("vocab", C.c_int),
                ("bytes_per_param", C.c_int), ("bytes_per_grad", C.c_int),
                ("bytes_per_os_per_param", C.c_int)]


class CostConfig(C.Structure):
    _fields_ = [("bucket_size", C.c_uint64), ("activation_mode", C.c_int),
                ("activation_coeff_full", C.c_double),
                ("activation_coeff_recompute", C.c_double),
                ("tmp_in_flight_buckets", C.c_int), ("tmp_include_gather_buffer", C.c_int),
                ("exact_residual_buckets", C.c_int), ("flops_coeff_param", C.c_double),
                ("flops_coeff_attn", C.c_double)]


class TimeBreakdown(C.Structure):
    _fields_ = [(n, C.c_double) for n in
                ("t_p", "t_g", "t_os_allreduce", "t_os_broadcast", "total")]


class MemoryBreakdown(C.Structure):
    _fields_ = [(n, C.c_double) for n in
                ("d_params", "d_grads", "d_os", "d_modelstate", "d_activation", "d_tmp",
                 "d_total")]


class StepRoofline(C.Structure):
    _fields_ = [("owned", C.c_uint64), ("hbm_bytes", C.c_uint64),
                ("nvlink_in_bytes", C.c_uint64), ("nvlink_out_bytes", C.c_uint64),
                ("t_hbm", C.c_double), ("t_nvlink", C.c_double), ("t_step", C.c_double)]


class PlanResult(C.Structure):
    _fields_ = [("plan", Plan), ("time", TimeBreakdown), ("memory", MemoryBreakdown),
                ("feasible", C.c_int), ("rank", C.c_int)]


class SimConfig(C.Structure):
    _fields_ = [("overlap_tier", C.c_int), ("recompute", C.c_int),
                ("comm_streams", C.c_int), ("compute_time_source", C.c_int),
                ("peak_flops_per_gpu", C.c_double), ("compute_efficiency", C.c_double),
                ("fwd_times", C.POINTER(C.c_double)),
                ("bwd_grad_weight_times", C.POINTER(C.c_double)),
                ("bwd_grad_input_times", C.POINTER(C.c_double)),
                ("head_fwd_time", C.c_double), ("head_bwd_time", C.c_double)]


class EngineConfig(C.Structure):
    _fields_ = [("tensor_sizes", C.POINTER(C.c_uint64)), ("n_tensors", C.c_int),
                ("plan", Plan), ("dp_mesh", Mesh), ("rank", C.c_int), ("device", C.c_int),
                ("layout", C.c_int), ("lr", C.c_double), ("beta1", C.c_double),
                ("beta2", C.c_double), ("eps", C.c_double), ("weight_decay", C.c_double),
                ("seed", C.c_uint64), ("skip_gathers", C.c_int),
                ("micro_batches", C.c_int), ("grad_ring_elems", C.c_uint64)]


class EngineInfo(C.Structure):
    _fields_ = [("total_params", C.c_uint64), ("owned", C.c_uint64),
                ("n_segments", C.c_int), ("world", C.c_int), ("os_block", C.c_int),
                ("os_position", C.c_int), ("os_group_size", C.c_int),
                ("replica_count", C.c_int), ("ntiles", C.c_int), ("grid", C.c_int),
                ("block", C.c_int), ("grads", C.c_void_p), ("params", C.c_void_p),
                ("master", C.c_void_p), ("exp_avg", C.c_void_p),
                ("exp_avg_sq", C.c_void_p), ("device_bytes", C.c_uint64),
                ("sp", C.c_int), ("p_position", C.c_int), ("param_elems", C.c_uint64),
                ("n_units", C.c_int), ("slot_elems", C.c_uint64),
                ("variant", C.c_int), ("micro_batches", C.c_int), ("grad_shards", C.c_int),
                ("acc_elems", C.c_uint64), ("acc_sources", C.c_int),
                ("acc_holders", C.c_int), ("grad_elems", C.c_uint64),
                ("secondary_shards", C.c_int), ("secondary_elems", C.c_uint64)]


class SchedConfig(C.Structure):
    _fields_ = [("model", Model), ("cost", CostConfig), ("sim", SimConfig),
                ("comm_ctas", C.c_int), ("compute_ctas", C.c_int), ("time_scale", C.c_double),
                ("optimizer_overlap", C.c_int), ("compute_mode", C.c_int), ("tokens", C.c_int),
                ("gemm_sm_margin", C.c_int), ("gather_mode", C.c_int), ("bc_mode", C.c_int),
                ("optimizer_variant", C.c_int), ("reduce_mode", C.c_int),
                ("grad_source", C.c_int)]


class SchedInfo(C.Structure):
    _fields_ = [("n_events", C.c_int), ("n_compute", C.c_int), ("n_gather", C.c_int),
                ("n_reduce", C.c_int), ("n_buckets", C.c_int), ("n_barriers", C.c_int),
                ("stream_count", C.c_int), ("predicted_step_s", C.c_double),
                ("predicted_compute_s", C.c_double), ("mirrored_bc", C.c_int),
                ("grad_ring_need", C.c_uint64)]


P = C.POINTER
vp = C.c_void_p
u64 = C.c_uint64

# name -> (restype, argtypes)
SIGNATURES = {
    "amsp_abi_version": (C.c_int, []),
    "amsp_last_error": (C.c_char_p, []),
    "amsp_cost_config_default": (None, [P(CostConfig)]),
    "amsp_sim_config_default": (None, [P(SimConfig)]),
    "amsp_profile_synthetic": (C.c_int, [C.c_double, C.c_double, C.c_double, C.c_double,
                                         P(Mesh), C.c_int, P(u64), C.c_int, P(vp)]),
    "amsp_profile_from_csv": (C.c_int, [C.c_char_p, P(vp)]),
    "amsp_profile_from_json": (C.c_int, [C.c_char_p, P(vp)]),
    "amsp_profile_load": (C.c_int, [C.c_char_p, P(vp)]),
    "amsp_profile_to_json": (C.c_int, [vp, C.c_char_p, C.c_size_t, P(C.c_size_t)]),
    "amsp_collective_time": (C.c_int, [vp, C.c_int, u64, Mesh, P(C.c_double)]),
    "amsp_profile_free": (None, [vp]),
    "amsp_ring_time": (C.c_int, [C.c_int, C.c_double, C.c_int, C.c_double, C.c_double,
                                 P(C.c_double)]),
    "amsp_validate_plan": (C.c_int, [P(Plan), P(Cluster), P(C.c_int), C.c_char_p,
                                     C.c_size_t]),
    "amsp_preset": (C.c_int, [C.c_char_p, P(Cluster), P(Plan)]),
    "amsp_memory_breakdown": (C.c_int, [P(Model), P(Plan), P(CostConfig),
                                        P(MemoryBreakdown)]),
    "amsp_total_comm_time": (C.c_int, [P(Model), P(Cluster), P(Plan), vp, P(CostConfig),
                                       P(TimeBreakdown)]),
    "amsp_grad_bucket_count": (C.c_int, [P(Model), P(Plan), P(CostConfig), P(u64)]),
    "amsp_partition_greedy": (C.c_int, [P(u64), C.c_int, C.c_int, P(C.c_int), P(u64)]),
    "amsp_enumerate_candidates": (C.c_int, [P(Cluster), P(Plan), C.c_int, P(C.c_int)]),
    "amsp_solve": (C.c_int, [P(Model), P(Cluster), vp, P(CostConfig), P(PlanResult),
                             P(u64), P(u64), P(PlanResult), C.c_int, P(C.c_int)]),
    "amsp_simulate": (C.c_int, [P(Model), P(Cluster), P(Plan), vp, P(CostConfig),
                                P(SimConfig), P(C.c_double), P(C.c_double), P(C.c_int),
                                C.c_char_p, C.c_size_t, P(C.c_size_t)]),
    "amsp_layout_segments": (C.c_int, [P(u64), C.c_int, C.c_int, C.c_int, C.c_int, P(u64),
                                       P(u64), P(u64), C.c_int, P(C.c_int), P(u64)]),
    "amsp_mesh_group": (C.c_int, [Mesh, Mesh, C.c_int, P(C.c_int), P(C.c_int), P(C.c_int),
                                  C.c_int, P(C.c_int)]),
    "amsp_pshard_layout": (C.c_int, [P(u64), C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                     C.c_int, P(u64), P(u64), P(u64), P(u64), C.c_int,
                                     P(C.c_int), P(u64)]),
    "amsp_step_roofline": (C.c_int, [P(u64), C.c_int, P(Plan), Mesh, C.c_int, C.c_int, C.c_int,
                                     C.c_double, C.c_double, P(C.c_int), P(StepRoofline)]),
    "amsp_model_tensors": (C.c_int, [P(Model), P(u64), C.c_int, P(C.c_int)]),
    "amsp_solve_roofline": (C.c_int, [P(Model), P(Cluster), vp, P(CostConfig), C.c_double,
                                      C.c_double, C.c_int, P(PlanResult), P(StepRoofline),
                                      P(PlanResult), P(StepRoofline), C.c_int, P(C.c_int)]),
    "amsp_engine_create": (C.c_int, [P(EngineConfig), P(vp)]),
    "amsp_engine_info": (C.c_int, [vp, P(EngineInfo)]),
    "amsp_engine_export_handle": (C.c_int, [vp, vp]),
    "amsp_engine_import_handles": (C.c_int, [vp, vp, C.c_int]),
    "amsp_engine_unit": (C.c_int, [vp, C.c_int, P(C.c_int), P(C.c_int), P(u64)]),
    "amsp_engine_gather": (C.c_int, [vp, C.c_int, C.c_int, vp]),
    "amsp_engine_gather_secondary": (C.c_int, [vp, C.c_int, C.c_int, vp]),
    "amsp_engine_link_local": (C.c_int, [P(vp), C.c_int]),
    "amsp_engine_link_local_sync": (C.c_int, [P(vp), C.c_int]),
    "amsp_sched_barrier_owner": (C.c_int, [vp, C.c_int, P(C.c_int), P(C.c_int), P(C.c_int)]),
    "amsp_engine_init_state": (C.c_int, [vp, vp]),
    "amsp_engine_synth_grads": (C.c_int, [vp, C.c_int, vp]),
    "amsp_engine_synth_grads_mb": (C.c_int, [vp, C.c_int, C.c_int, vp]),
    "amsp_engine_accumulate": (C.c_int, [vp, C.c_int, C.c_int, vp]),
    "amsp_engine_accum_ms": (C.c_int, [vp, C.POINTER(C.c_double), C.POINTER(C.c_int)]),
    "amsp_engine_nvlink_probe": (C.c_int, [vp, C.c_uint64, C.c_int, C.c_int,
                                           C.POINTER(C.c_double)]),
    "amsp_engine_step": (C.c_int, [vp, C.c_int, vp]),
    "amsp_engine_step_host": (C.c_int, [vp, C.c_int, vp, P(C.c_float), vp]),
    "amsp_engine_stats": (C.c_int, [vp, P(C.c_float)]),
    "amsp_engine_read": (C.c_int, [vp, C.c_int, u64, u64, vp]),
    "amsp_engine_write": (C.c_int, [vp, C.c_int, u64, u64, vp]),
    "amsp_engine_launch_count": (C.c_int, [vp, P(u64)]),
    "amsp_engine_tune": (C.c_int, [vp, C.c_int, C.c_int]),
    "amsp_engine_tune_gather": (C.c_int, [vp, C.c_int]),
    "amsp_engine_time_kernel": (C.c_int, [vp, C.c_int]),
    "amsp_engine_kernel_ms": (C.c_int, [vp, P(C.c_double), P(C.c_int)]),
    "amsp_engine_gather_ms": (C.c_int, [vp, P(C.c_double), P(C.c_int)]),
    "amsp_engine_destroy": (None, [vp]),
    "amsp_sched_create": (C.c_int, [vp, P(SchedConfig), vp, P(vp)]),
    "amsp_sched_info": (C.c_int, [vp, P(SchedInfo)]),
    "amsp_sched_step": (C.c_int, [vp, C.c_int, vp, C.c_int]),
    "amsp_sched_enable_trace": (C.c_int, [vp, C.c_int]),
    "amsp_sched_flush": (C.c_int, [vp, vp]),
    "amsp_sched_trace": (C.c_int, [vp, C.c_char_p, C.c_size_t, P(C.c_size_t), P(C.c_double)]),
    "amsp_sched_predicted_trace": (C.c_int, [vp, C.c_char_p, C.c_size_t, P(C.c_size_t)]),
    "amsp_sched_destroy": (None, [vp]),
    "amsp_k_synth_grad": (C.c_int, [vp, u64, u64, u64, C.c_int, C.c_int, vp]),
    "amsp_k_adamw": (C.c_int, [vp, C.c_int, vp, vp, vp, vp, u64, C.c_int, C.c_double,
                               C.c_double, C.c_double, C.c_double, C.c_double, C.c_double,
                               vp]),
    "amsp_k_upcast_scale": (C.c_int, [vp, vp, u64, C.c_float, vp]),
    "amsp_k_spin": (C.c_int, [C.c_int, u64, vp]),
    "amsp_k_rs_upcast_scale": (C.c_int, [P(vp), C.c_int, u64, vp, u64, C.c_float, vp]),
    "amsp_k_ag_downcast": (C.c_int, [vp, u64, P(vp), C.c_int, u64, vp]),
}

_lib: C.CDLL | None = None


def lib() -> C.CDLL:
    """Load libamsp.so (once). Raises if it has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise ImportError(
            f"{LIB_PATH} is missing: run `python -m paper_2311_00257_b200.build` "
            "(or __graft_entry__.build()); there is no fallback implementation")
    L = C.CDLL(str(LIB_PATH), mode=os.RTLD_NOW | os.RTLD_GLOBAL)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    if L.amsp_abi_version() != 2:
        raise ImportError("libamsp.so ABI version mismatch")
    _lib = L
    return L


def check(code: int) -> None:
    if code == AMSP_OK:
        return
    msg = (lib().amsp_last_error() or b"").decode(errors="replace")
    cls = {AMSP_EINVAL: InvalidConfig, AMSP_EINFEASIBLE: Infeasible,
           AMSP_ECUDA: CudaError}.get(code, AmspError)
    raise cls(code, msg)
