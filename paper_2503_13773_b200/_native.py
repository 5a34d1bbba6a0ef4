"""ctypes binding of include/cacheopt.h (the in-tree libcacheopt.so).

There is no CPU fallback: if the shared library is missing or cannot be
loaded, importing the engine raises immediately.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

LIB_PATH = Path(__file__).resolve().parent / "_lib" / "libcacheopt.so"

CO_OK, CO_EINVAL, CO_ECUDA, CO_EDEVICE = 0, 1, 2, 3
MAX_SLO_EDGES = 8
NSTAGES = 8
STAGES = ("begin+admit", "classify", "bucket", "plan", "apply", "check", "data", "decode")

EV_ARRIVE, EV_ADMIT, EV_ITER, EV_PREEMPT, EV_READMIT, EV_COMPLETE = range(6)
CO_EAGAIN = 4  # co_drain_log: buffers too small, sizes returned
CAUSES = ("plan", "squeeze", "collision")

FIELDS = ("STATE GENERATED USED KV_NEED PREFILL_DONE PREEMPTION_COUNT PREEMPTION_TIME "
          "FIRST_TOKEN LAST_TOKEN MAX_TBT READY_AT PREEMPT_STARTED SWAP_OUT_DONE LAST_STRATEGY "
          "FIRST_START COMPLETION ALLOCATED_KVC PREDICTED ESTIMATED HOLDS GRANTED HOST "
          "EMBED_OFFSET RESERVED_DRAWN RECORD_SEQ CLAIM_WAITER SORTED_ORDER").split()
FIELD = {name: k for k, name in enumerate(FIELDS)}

I64P = C.POINTER(C.c_int64)
I32P = C.POINTER(C.c_int32)
U8P = C.POINTER(C.c_uint8)


class CoConfig(C.Structure):
    _fields_ = [
        ("capacity_tokens", C.c_int64), ("reserved_blocks", C.c_int32), ("allow_stacking", C.c_int32),
        ("block_size", C.c_int32), ("buffer_b", C.c_int32), ("token_budget", C.c_int32),
        ("preallocate_m", C.c_int32), ("decode_runway_iters", C.c_int32), ("victim_rule_fcfs", C.c_int32),
        ("epsilon_us", C.c_int64), ("n_slo_edges", C.c_int32), ("token_step", C.c_int32),
        ("slo_edges_us", C.c_int64 * MAX_SLO_EDGES), ("iter_base_ms", C.c_double),
        ("iter_per_token_ms", C.c_double), ("horizon_factor", C.c_int64), ("validate_every", C.c_int32),
        ("record_events", C.c_int32), ("padding", C.c_int32), ("invert_amortization", C.c_int32), ("s_star", C.c_int64),
        ("t_i_init_us", C.c_int64), ("kv_layers", C.c_int32), ("kv_heads", C.c_int32), ("q_heads", C.c_int32),
        ("head_dim", C.c_int32), ("host_swap_pages", C.c_int64), ("decode", C.c_int32), ("decode_split", C.c_int32),
        ("policy", C.c_int32), ("vllm_block_tokens", C.c_int32), ("s3_bucket_tokens", C.c_int32),
        ("rlp_padding", C.c_int32),
    ]


POLICY_CODE = {"cacheopt": 0, "vllm_block": 1, "sarathi_chunked": 2, "rlp": 3, "s3": 4}


class CoTrace(C.Structure):
    _fields_ = [
        ("n", C.c_int64), ("req_id", I64P), ("arrival_us", I64P), ("prompt_len", I32P),
        ("true_output_len", I32P), ("slo_ttft_us", I64P), ("slo_tbt_us", I64P), ("err_draw", I32P),
        ("flip_draw", U8P),
    ]


class CoLuts(C.Structure):
    _fields_ = [("s_max", C.c_int64), ("swap_half_us", I64P), ("recompute_us", I64P),
                ("survive_swap_us", I64P), ("survive_rec_us", I64P)]


class CoScalars(C.Structure):
    _fields_ = [
        ("now_us", C.c_int64), ("horizon_us", C.c_int64), ("first_arrival_us", C.c_int64),
        ("t_i_max_us", C.c_int64), ("footprint_tokens", C.c_int64), ("granted_tokens", C.c_int64),
        ("used_tokens", C.c_int64), ("generated_total", C.c_int64), ("iterations", C.c_int64),
        ("steps", C.c_int64), ("record_seq", C.c_int64), ("n_events", C.c_int64), ("n_samples", C.c_int64),
        ("decisions", C.c_int64),
        ("reserved_blocks_current", C.c_int32), ("n_live", C.c_int32), ("n_pending", C.c_int32),
        ("done", C.c_int32), ("stalled", C.c_int32), ("last_step_result", C.c_int32), ("error", C.c_int32),
        ("_pad0", C.c_int32),
    ]


class CoStepArgs(C.Structure):  # include/cacheopt.h co_step_args
    _fields_ = [("eng", C.c_void_p), ("result", C.c_void_p), ("members", C.c_void_p), ("max_members", C.c_int64),
                ("n_members", C.c_void_p), ("iter_end_us", C.c_void_p), ("events", C.c_void_p),
                ("max_events", C.c_int64), ("log_members", C.c_void_p), ("max_log_members", C.c_int64),
                ("samples", C.c_void_p), ("max_samples", C.c_int64), ("counts", C.c_void_p), ("drain", C.c_int32),
                ("_pad", C.c_int32), ("ids", C.c_void_p), ("members_ids", C.c_void_p)]


class CoEvent(C.Structure):
    _fields_ = [("kind", C.c_int32), ("idx", C.c_int32), ("t", C.c_int64), ("a", C.c_int64),
                ("b", C.c_int64), ("c", C.c_int64)]


EXPORTS = (
    "co_create", "co_destroy", "co_step", "co_run", "co_preempt", "co_get_scalars", "co_read_field",
    "co_drain_events", "co_pending_events", "co_pending_log", "co_drain_log", "co_step_result_log", "co_step_packed", "co_pool_create", "co_pool_destroy", "co_pool_op", "co_pool_find_host",
    "co_pool_state", "co_pool_check", "co_pool_read_tables", "co_sched_op", "co_swap_io_stats", "co_plan_snapshot", "co_drain_samples", "co_read_token_times",
    "co_check_invariants", "co_last_device_ms", "co_kernels_per_step", "co_time_steps", "co_last_error",
    "co_version", "co_read_block_tables", "co_data_stats", "co_kv_verify", "co_read_decode", "co_host_link_gbs",
    "co_set_decode", "co_swap_bench", "co_nccl_unique_id", "co_attach_nccl", "co_global_reserve",
    "co_phase_profile", "co_step_result", "co_prepare_step", "co_metrics", "co_pcg64_seed", "co_gen_raw", "co_gen_std",
    "co_gen_trace", "co_gen_slos", "co_gen_predictor",
)

_lib = None


class CoMetricsRaw(C.Structure):
    _fields_ = [(k, C.c_int64) for k in ("completed", "ok_ttft", "ok_tbt", "generated", "preemption_total",
                                         "preempted", "sum_ttft", "sum_gap", "sum_wait", "sum_exec", "sum_pdec",
                                         "sum_ptime")] + [
        ("count", C.c_int64 * 4), ("norm_sum", C.c_double), ("order_stat", (C.c_double * 7) * 4)]


class CoTraceSpec(C.Structure):
    _fields_ = [("n", C.c_int64), ("gap_scale", C.c_double), ("mu_in", C.c_double), ("sigma_in", C.c_double),
                ("mu_out", C.c_double), ("sigma_out", C.c_double), ("input_min", C.c_int32),
                ("input_max", C.c_int32), ("output_min", C.c_int32), ("output_max", C.c_int32)]


class CoSloSpec(C.Structure):
    _fields_ = [("base_ttft_us", C.c_int64), ("base_tbt_us", C.c_int64), ("scale_lo", C.c_double),
                ("scale_hi", C.c_double), ("chunk_budget", C.c_int32), ("_pad", C.c_int32)]


class CoPredictorSpec(C.Structure):
    _fields_ = [("error_dist", C.c_int32), ("_pad", C.c_int32), ("error_scale", C.c_double),
                ("direction_accuracy", C.c_double)]


ERR_DIST = {"zero": 0, "uniform": 1, "normal": 2}


class NativeError(RuntimeError):
    pass


def load() -> C.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    path = os.environ.get("CACHEOPT_LIB", str(LIB_PATH))
    if not os.path.exists(path):
        raise NativeError(f"libcacheopt.so not built at {path}: run __graft_entry__.build()")
    lib = C.CDLL(path)
    V = C.c_void_p
    sig = {
        "co_create": (C.c_int, [C.POINTER(CoConfig), C.POINTER(CoTrace), C.POINTER(CoLuts), C.c_int,
                                C.POINTER(V)]),
        "co_destroy": (C.c_int, [V]),
        "co_step": (C.c_int, [V, I32P]),
        "co_prepare_step": (C.c_int, [V]),
        "co_run": (C.c_int, [V, C.c_int64, C.c_int32, I64P]),
        "co_preempt": (C.c_int, [V, C.c_int64, C.c_int32, C.c_int64, C.c_int32]),
        "co_get_scalars": (C.c_int, [V, C.POINTER(CoScalars)]),
        "co_read_field": (C.c_int, [V, C.c_int32, I64P]),
        "co_drain_events": (C.c_int, [V, C.POINTER(CoEvent), C.c_int64, I32P, C.c_int64, I64P, I64P]),
        "co_pending_events": (C.c_int, [V, I64P, I64P]),
        "co_pending_log": (C.c_int, [V, I64P]),
        "co_pool_create": (C.c_int, [C.c_int64, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                                     C.POINTER(V)]),
        "co_pool_destroy": (C.c_int, [V]),
        "co_pool_op": (C.c_int, [V, C.c_int32, C.c_int32, C.c_int64, C.c_int64, C.c_int64, I64P]),
        "co_pool_find_host": (C.c_int, [V, C.c_int32, I64P, C.c_int64, C.c_int64, C.c_int64, I64P]),
        "co_pool_state": (C.c_int, [V, I64P, I64P]),
        "co_pool_check": (C.c_int, [V]),
        "co_sched_op": (C.c_int, [C.c_int32, C.c_int32, I64P, I64P, I64P, C.c_int32]),
        "co_swap_io_stats": (C.c_int, [V, I64P]),
        "co_plan_snapshot": (C.c_int, [V, I64P, I64P, I64P, I32P, C.c_int64]),
        "co_pool_read_tables": (C.c_int, [V, I32P, I32P, C.c_int64, I32P, I32P]),
        "co_drain_log": (C.c_int, [V, V, C.c_int64, V, C.c_int64, V, C.c_int64, V]),
        "co_step_result_log": (C.c_int, [V, V, V, C.c_int64, V, V, V, C.c_int64, V, C.c_int64, V, C.c_int64, V]),
        "co_step_packed": (C.c_int, [V]),
        "co_drain_samples": (C.c_int, [V, I64P, C.c_int64, I64P]),
        "co_read_token_times": (C.c_int, [V, I64P, I64P]),
        "co_check_invariants": (C.c_int, [V]),
        "co_last_device_ms": (C.c_int, [V, C.POINTER(C.c_double)]),
        "co_kernels_per_step": (C.c_int, [V, I32P]),
        "co_time_steps": (C.c_int, [V, C.c_int32, C.c_int64, C.POINTER(C.c_double), C.POINTER(C.c_double)]),
        "co_read_block_tables": (C.c_int, [V, I32P, I32P, C.c_int64, I32P, I32P]),
        "co_data_stats": (C.c_int, [V, I64P]),
        "co_kv_verify": (C.c_int, [V, I64P, I64P]),
        "co_read_decode": (C.c_int, [V, I32P, I32P, C.POINTER(C.c_float), C.c_int64, I64P, I64P]),
        "co_host_link_gbs": (C.c_int, [C.c_int64, C.POINTER(C.c_double), C.POINTER(C.c_double)]),
        "co_set_decode": (C.c_int, [V, C.c_int32]),
        "co_swap_bench": (C.c_int, [V, C.c_int64, C.c_int32, C.POINTER(C.c_double), C.POINTER(C.c_double)]),
        "co_nccl_unique_id": (C.c_int, [U8P]),
        "co_attach_nccl": (C.c_int, [V, U8P, C.c_int32, C.c_int32]),
        "co_global_reserve": (C.c_int, [V, I64P, I64P]),
        "co_phase_profile": (C.c_int, [V, C.c_int32, I64P]),
        "co_step_result": (C.c_int, [V, I32P, I32P, C.c_int64, I64P, I64P]),
        "co_metrics": (C.c_int, [V, C.POINTER(CoMetricsRaw)]),
        "co_pcg64_seed": (C.c_int, [C.POINTER(C.c_uint64), C.c_int32, C.POINTER(C.c_uint64)]),
        "co_gen_raw": (C.c_int, [C.c_uint64, C.c_uint64, C.c_int64, C.c_int, V]),
        "co_gen_std": (C.c_int, [C.c_int32, C.c_uint64, C.c_uint64, C.c_int64, C.c_int, V]),
        "co_gen_trace": (C.c_int, [C.POINTER(CoTraceSpec), C.c_uint64, C.c_int, V, V, V]),
        "co_gen_slos": (C.c_int, [C.c_int64, V, C.POINTER(CoSloSpec), C.c_uint64, C.c_int, V, V]),
        "co_gen_predictor": (C.c_int, [C.c_int64, C.POINTER(CoPredictorSpec), C.c_uint64, C.c_int, V, V]),
        "co_last_error": (C.c_char_p, []),
        "co_version": (C.c_char_p, []),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(rc: int, what: str) -> None:
    if rc != CO_OK:
        msg = _lib.co_last_error().decode() if _lib is not None else ""
        kind = {CO_EINVAL: ValueError, CO_EDEVICE: RuntimeError}.get(rc, NativeError)
        raise kind(f"{what}: {msg}")
