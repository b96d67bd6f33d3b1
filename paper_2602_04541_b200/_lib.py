"""ctypes binding of the in-tree C-ABI library ``liblyc.so`` (include/lyc.h).

The library is the product: there is no Python or CPU fallback.  If the
shared object is missing the import fails loudly with the build command.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

LIB_PATH = Path(__file__).resolve().parent / "liblyc.so"

LYC_OK, LYC_EINVAL, LYC_ESTATE, LYC_ECUDA, LYC_ENOTSUP, LYC_ENCCL = 0, -1, -2, -3, -4, -5
DTYPE_F32, DTYPE_BF16 = 0, 1
POLICY_TOPK, POLICY_TOPP, POLICY_THRESHOLD, POLICY_RATIO = 0, 1, 2, 3
SELECT_TOKENS, SELECT_BLOCKS, SELECT_NONE = 0, 1, 2

# Exported symbols (must match include/lyc.h; checked by tests/test_abi.py).
SYMBOLS = [
    "lyc_last_error", "lyc_version", "lyc_launch_count", "lyc_plan_splits", "lyc_latency_model",
    "lyc_fraction_budget", "lyc_workload_run", "lyc_args_top_k", "lyc_decoder_create",
    "lyc_decoder_destroy", "lyc_decoder_step", "lyc_decoder_layer", "lyc_decoder_capture",
    "lyc_decoder_replay", "lyc_decoder_index_cache", "lyc_decoder_launches_per_step",
    "lyc_decoder_step_bytes", "lyc_decoder_layer_attn_bytes", "lyc_decoder_set_timing",
    "lyc_decoder_attn_ms", "lyc_decoder_is_fused", "lyc_decoder_set_trace", "lyc_decoder_trace",
    "lyc_shard_layer", "lyc_shard_merge", "lyc_kv_write", "lyc_window_workspace",
    "lyc_window_attention", "lyc_decoder_step_varlen", "lyc_decoder_capture_varlen",
    "lyc_decoder_set_trace_sets", "lyc_decoder_traced_sets", "lyc_decoder_step_dev",
    "lyc_decoder_capture_dev", "lyc_decoder_status", "lyc_decoder_tune", "lyc_kv_append_dev",
    "lyc_plan_selftest", "lyc_decoder_refresh_sets", "lyc_decoder_sync_sets", "lyc_gemv",
]

GEMV_STORE, GEMV_RESIDUAL, GEMV_SILU_BF16, GEMV_QKV_ROPE = 0, 1, 2, 3
GEMV_FLAG_NEXT_IS_GEMV = 1

TUNE_RING_STAGES, TUNE_PER_LAYER_KERNELS, TUNE_PDL, TUNE_DEFER_SELECTION = 1, 2, 3, 4


class LycError(RuntimeError):
    code = None


class InvalidArgument(LycError, ValueError):
    """std::invalid_argument in the reference."""


class LogicError(LycError):
    """std::logic_error in the reference."""


class CudaError(LycError):
    pass


class NotSupported(LycError):
    pass


class lyc_workload(C.Structure):
    _fields_ = [
        ("batch", C.c_int64), ("n_kv_heads", C.c_int64), ("group_size", C.c_int64),
        ("d_head", C.c_int64), ("seq_len", C.c_int64), ("block_size", C.c_int64),
        ("kv_row_stride", C.c_int64), ("scale", C.c_float), ("dtype", C.c_int32),
        ("k", C.c_void_p), ("v", C.c_void_p), ("q", C.c_void_p),
        ("blk_off", C.c_void_p), ("blk_ids", C.c_void_p),
    ]


class lyc_decode_config(C.Structure):
    _fields_ = [
        ("n_layers", C.c_int32), ("batch", C.c_int32), ("n_kv_heads", C.c_int32),
        ("group_size", C.c_int32), ("d_head", C.c_int32), ("dtype", C.c_int32),
        ("seq_cap", C.c_int64), ("policy_kind", C.c_int32), ("select_mode", C.c_int32),
        ("top_k", C.c_int64), ("ratio", C.c_double), ("block_size", C.c_int32),
        ("num_splits", C.c_int32), ("scale", C.c_float), ("roles", C.c_void_p),
    ]


class lyc_kv_layout(C.Structure):
    _fields_ = [
        ("n_layers", C.c_int32), ("batch", C.c_int32), ("n_kv_heads", C.c_int32),
        ("d_head", C.c_int32), ("dtype", C.c_int32), ("pad", C.c_int32), ("seq_cap", C.c_int64),
    ]


class lyc_gemv_desc(C.Structure):
    _fields_ = [
        ("M", C.c_int64), ("K", C.c_int64), ("w", C.c_void_p), ("x", C.c_void_p),
        ("xb", C.c_void_p), ("gain", C.c_void_p), ("eps", C.c_float), ("mode", C.c_int32),
        ("y", C.c_void_p), ("yb", C.c_void_p), ("q_out", C.c_void_p), ("k_cache", C.c_void_p),
        ("v_cache", C.c_void_p), ("slab_stride", C.c_int64), ("nq", C.c_int32),
        ("nkv", C.c_int32), ("d", C.c_int32), ("flags", C.c_int32), ("pos", C.c_int64),
        ("prefetch", C.c_void_p), ("prefetch_bytes", C.c_int64),
    ]


_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`"
            " (or make -C paper_2602_04541_b200/csrc).  There is no CPU fallback.")
    L = C.CDLL(str(LIB_PATH))
    vp, i64, i32, dbl = C.c_void_p, C.c_int64, C.c_int32, C.c_double
    L.lyc_last_error.restype = C.c_char_p
    L.lyc_version.restype = C.c_char_p
    L.lyc_launch_count.restype = i64
    L.lyc_plan_splits.restype = i64
    L.lyc_plan_splits.argtypes = [i64, i64, vp, i64, vp, vp, vp, i64]
    L.lyc_latency_model.restype = C.c_int
    L.lyc_latency_model.argtypes = [i64, i64, vp, i64, i64, vp, vp]
    L.lyc_fraction_budget.restype = i64
    L.lyc_fraction_budget.argtypes = [dbl, i64]
    L.lyc_workload_run.restype = C.c_int
    L.lyc_workload_run.argtypes = [C.POINTER(lyc_workload), i64, vp, vp, vp]
    L.lyc_args_top_k.restype = i64
    L.lyc_args_top_k.argtypes = [vp, i64, i64, vp, vp]
    L.lyc_decoder_create.restype = C.c_int
    L.lyc_decoder_create.argtypes = [C.POINTER(lyc_decode_config), C.POINTER(vp)]
    L.lyc_decoder_destroy.restype = C.c_int
    L.lyc_decoder_destroy.argtypes = [vp]
    L.lyc_decoder_step.restype = C.c_int
    L.lyc_decoder_step.argtypes = [vp, vp, vp, vp, i64, vp, vp]
    L.lyc_decoder_step_varlen.restype = C.c_int
    L.lyc_decoder_step_varlen.argtypes = [vp, vp, vp, vp, C.POINTER(C.c_int64), vp, vp]
    L.lyc_decoder_capture_varlen.restype = C.c_int
    L.lyc_decoder_capture_varlen.argtypes = [vp, vp, vp, vp, C.POINTER(C.c_int64), vp, vp]
    L.lyc_decoder_layer.restype = C.c_int
    L.lyc_decoder_layer.argtypes = [vp, i32, vp, vp, vp, i64, vp, vp]
    L.lyc_gemv.restype = C.c_int
    L.lyc_gemv.argtypes = [C.POINTER(lyc_gemv_desc), vp]
    L.lyc_decoder_sync_sets.restype = C.c_int
    L.lyc_decoder_sync_sets.argtypes = [vp, vp]
    L.lyc_decoder_refresh_sets.restype = C.c_int
    L.lyc_decoder_refresh_sets.argtypes = [vp, i32, vp, vp, i64, vp]
    L.lyc_decoder_capture.restype = C.c_int
    L.lyc_decoder_capture.argtypes = [vp, vp, vp, vp, i64, vp, vp]
    L.lyc_decoder_replay.restype = C.c_int
    L.lyc_decoder_replay.argtypes = [vp, vp]
    L.lyc_decoder_index_cache.restype = C.c_int
    L.lyc_decoder_index_cache.argtypes = [vp, C.POINTER(vp), C.POINTER(vp), C.POINTER(i64)]
    L.lyc_decoder_launches_per_step.restype = i64
    L.lyc_decoder_launches_per_step.argtypes = [vp, i64]
    L.lyc_decoder_step_bytes.restype = i64
    L.lyc_decoder_step_bytes.argtypes = [vp, i64]
    L.lyc_decoder_layer_attn_bytes.restype = i64
    L.lyc_decoder_layer_attn_bytes.argtypes = [vp, i32, i64]
    L.lyc_decoder_set_timing.restype = C.c_int
    L.lyc_decoder_set_timing.argtypes = [vp, C.c_int]
    L.lyc_decoder_attn_ms.restype = C.c_int
    L.lyc_decoder_attn_ms.argtypes = [vp, vp]
    L.lyc_decoder_is_fused.restype = C.c_int
    L.lyc_decoder_is_fused.argtypes = [vp]
    L.lyc_decoder_set_trace.restype = C.c_int
    L.lyc_decoder_set_trace.argtypes = [vp, C.c_int]
    L.lyc_decoder_trace.restype = i64
    L.lyc_decoder_trace.argtypes = [vp, vp, i64]
    L.lyc_decoder_set_trace_sets.restype = C.c_int
    L.lyc_decoder_set_trace_sets.argtypes = [vp, C.c_int]
    L.lyc_decoder_traced_sets.restype = i64
    L.lyc_decoder_traced_sets.argtypes = [vp, vp, vp, i64]
    L.lyc_decoder_step_dev.restype = C.c_int
    L.lyc_decoder_step_dev.argtypes = [vp, vp, vp, vp, vp, vp, vp]
    L.lyc_decoder_capture_dev.restype = C.c_int
    L.lyc_decoder_capture_dev.argtypes = [vp, vp, vp, vp, vp, vp, vp]
    L.lyc_decoder_status.restype = C.c_int
    L.lyc_decoder_status.argtypes = [vp, vp]
    L.lyc_decoder_tune.restype = C.c_int
    L.lyc_decoder_tune.argtypes = [vp, i32, i64]
    L.lyc_kv_append_dev.restype = C.c_int
    L.lyc_kv_append_dev.argtypes = [vp, vp, C.POINTER(lyc_kv_layout), i32, vp, vp, vp, vp]
    L.lyc_plan_selftest.restype = C.c_int
    L.lyc_plan_selftest.argtypes = [C.POINTER(lyc_decode_config), i64, C.POINTER(C.c_int64), i32]
    L.lyc_shard_layer.restype = C.c_int
    L.lyc_shard_layer.argtypes = [vp, i32, vp, vp, vp, i64, i64, vp, vp, vp, vp, vp]
    L.lyc_shard_merge.restype = C.c_int
    L.lyc_shard_merge.argtypes = [vp, i32, i32, vp, vp, vp, vp, i64, i64, i64, i64, vp, vp, vp]
    L.lyc_kv_write.restype = C.c_int
    L.lyc_kv_write.argtypes = [vp, vp, C.POINTER(lyc_kv_layout), i32, i64, i64, vp, vp, vp]
    L.lyc_window_workspace.restype = C.c_int64
    L.lyc_window_workspace.argtypes = [C.POINTER(lyc_kv_layout), i32, i32]
    L.lyc_window_attention.restype = C.c_int
    L.lyc_window_attention.argtypes = [C.POINTER(lyc_kv_layout), i32, vp, vp, i32, C.c_float, i64,
                                       i32, vp, vp, vp, i64, vp]
    _lib = L
    return L


def check(rc: int) -> int:
    """Map a C-ABI status to the reference's exception types."""
    if rc >= 0:
        return rc
    msg = lib().lyc_last_error().decode(errors="replace")
    exc = {LYC_EINVAL: InvalidArgument, LYC_ESTATE: LogicError, LYC_ECUDA: CudaError,
           LYC_ENOTSUP: NotSupported}.get(rc, LycError)
    e = exc(msg or f"lyc error {rc}")
    e.code = rc
    raise e
