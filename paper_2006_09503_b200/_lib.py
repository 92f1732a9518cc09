"""ctypes binding of libp2bw.so (include/p2bw.h).

The shared library is built in-tree by ``paper_2006_09503_b200.build``.  There
is no fallback: if the library is missing or fails to load, every entry point
raises, so no caller can silently run something other than the CUDA engine.
"""
from __future__ import annotations

import ctypes as C
import threading
from pathlib import Path

LIB_PATH = Path(__file__).resolve().parent / "libp2bw.so"

_lock = threading.Lock()
_lib: C.CDLL | None = None


class P2bwError(RuntimeError):
    """Raised for a nonzero p2bw_* status; the text is p2bw_last_error()
    (pipesim::Error wording, reference core/include/pipesim/error.hpp:9-12)."""


class GemmEpilogue(C.Structure):
    _fields_ = [
        ("kind", C.c_int),
        ("d", C.c_void_p),
        ("ldd", C.c_longlong),
        ("bias", C.c_void_p),
        ("residual", C.c_void_p),
        ("ldr", C.c_longlong),
        ("preact", C.c_void_p),
        ("gelu", C.c_int),
        ("aux", C.c_void_p),
        ("alpha", C.c_float),
        ("beta", C.c_float),
        ("workspace", C.c_void_p),
        ("workspace_floats", C.c_longlong),
        ("bias_grad", C.c_void_p),
        ("bias_grad_accumulate", C.c_int),
        ("bias_scratch", C.c_void_p),
        ("bias_scratch_floats", C.c_longlong),
    ]


class Op(C.Structure):
    _fields_ = [("kind", C.c_int), ("microbatch", C.c_int), ("weight_version", C.c_int)]


def _signatures():
    """(name, restype, argtypes) for every function include/p2bw.h declares."""
    i, ll, vp, sz, cp = C.c_int, C.c_longlong, C.c_void_p, C.c_size_t, C.c_char_p
    pi, pvp, psz = C.POINTER(C.c_int), C.POINTER(C.c_void_p), C.POINTER(C.c_size_t)
    return [
        ("p2bw_last_error", cp, []),
        ("p2bw_version", cp, []),
        ("p2bw_free", None, [vp]),
        ("p2bw_weight_version_2bw", i, [i, i, pi]),
        ("p2bw_required_versions", i, [i, i, i, pi]),
        ("p2bw_schedule_generate", i, [i, i, i, i, pvp]),
        ("p2bw_schedule_parse", i, [cp, pvp]),
        ("p2bw_schedule_num_stages", i, [vp, pi]),
        ("p2bw_schedule_ops", i, [vp, i, C.POINTER(C.POINTER(Op)), psz]),
        ("p2bw_schedule_serialize", i, [vp, pvp]),
        ("p2bw_schedule_destroy", None, [vp]),
        ("p2bw_policy_name", i, [i, C.POINTER(cp)]),
        ("p2bw_policy_parse", i, [cp, pi]),
        ("p2bw_plan", i, [cp, cp, ll, i, i, pvp]),
        ("p2bw_partition_equal", i, [cp, i, pvp]),
        ("p2bw_partition_balanced", i, [cp, i, i, pvp]),
        ("p2bw_engine_create", i, [vp, pvp]),
        ("p2bw_engine_destroy", None, [vp]),
        ("p2bw_engine_stage_weight_bytes", i, [vp, i, psz]),
        ("p2bw_engine_load_stage_weights", i, [vp, i, vp, sz]),
        ("p2bw_engine_init_weights", i, [vp]),
        ("p2bw_engine_set_data", i, [vp, vp, vp, i, i]),
        ("p2bw_engine_make_toy_data", i, [vp, i, i]),
        ("p2bw_engine_run", i, [vp, vp, vp, i]),
        ("p2bw_engine_run_schedule", i, [vp, i, i]),
        ("p2bw_engine_run_schedule_graph", i, [vp, i, i, C.POINTER(C.c_double)]),
        ("p2bw_engine_begin", i, [vp, i]),
        ("p2bw_engine_issue", i, [vp, i]),
        ("p2bw_engine_finish", i, [vp]),
        ("p2bw_engine_update_elapsed_ms", i, [vp, i, i, i, C.POINTER(C.c_double)]),
        ("p2bw_nccl_unique_id", i, [vp, sz]),
        ("p2bw_engine_join_replicas", i, [vp, vp, i, i]),
        ("p2bw_engine_export_replica", i, [vp, i, vp, sz]),
        ("p2bw_engine_join_replicas_ipc", i, [vp, i, vp, i, i]),
        ("p2bw_engine_is_local", i, [vp, i, C.POINTER(C.c_int)]),
        ("p2bw_engine_export_stage", i, [vp, i, vp, sz]),
        ("p2bw_engine_connect_stage", i, [vp, vp, sz]),
        ("p2bw_engine_sync", i, [vp]),
        ("p2bw_engine_set_trace", i, [vp, i]),
        ("p2bw_engine_trace_report", i, [vp, pvp]),
        ("p2bw_engine_counters", i, [vp, vp]),
        ("p2bw_engine_read_snapshot", i, [vp, i, i, vp, sz]),
        ("p2bw_engine_read_version", i, [vp, i, i, vp, sz]),
        ("p2bw_engine_read_master", i, [vp, i, vp, sz]),
        ("p2bw_engine_losses_async", i, [vp, i, i, vp]),
        ("p2bw_engine_losses", i, [vp, i, i, vp]),
        ("p2bw_profile_blocks", i, [vp, pi, i, i, i, cp, pvp]),
        ("p2bw_launch_count", ll, []),
        ("p2bw_profile_enable", None, [i]),
        ("p2bw_profile_collect", i, [vp, i, C.POINTER(C.c_int)]),
        ("p2bw_kernel_gemm_bf16", i, [vp, ll, i, vp, ll, i, i, i, i, C.POINTER(GemmEpilogue), vp]),
        ("p2bw_kernel_attention_fwd", i, [vp, vp, vp, i, i, i, i, vp]),
        ("p2bw_kernel_attention_bwd", i, [vp, vp, vp, vp, vp, vp, i, i, i, i, vp]),
        ("p2bw_kernel_attention_fwd_hd", i, [vp, vp, vp, i, i, i, i, i, vp]),
        ("p2bw_kernel_attention_bwd_hd", i, [vp, vp, vp, vp, vp, vp, i, i, i, i, i, vp]),
        ("p2bw_kernel_layernorm_fwd", i, [vp, vp, vp, vp, vp, vp, i, i, vp]),
        ("p2bw_kernel_layernorm_bwd", i, [vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, i, i, i, vp]),
        ("p2bw_kernel_softmax_xent", i, [vp, vp, i, i, i, C.c_float, vp, vp]),
        ("p2bw_kernel_colsum", i, [vp, i, i, i, vp, i, vp]),
        ("p2bw_debug_attention_timing", i, [vp]),
        ("p2bw_debug_gemm_timing", i, [vp]),
        ("p2bw_debug_gemm_plan", i, [i, i, i, i, i, i, i, C.POINTER(C.c_int)]),
    ]


def declared_symbols() -> list[str]:
    return [name for name, _, _ in _signatures()]


def _declare(lib: C.CDLL) -> None:
    for name, res, args in _signatures():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args


def lib() -> C.CDLL:
    global _lib
    with _lock:
        if _lib is None:
            if not LIB_PATH.exists():
                raise P2bwError(
                    f"{LIB_PATH} is missing: build it with `python -m paper_2006_09503_b200.build` "
                    "(there is no CPU fallback)")
            handle = C.CDLL(str(LIB_PATH), mode=C.RTLD_GLOBAL)
            _declare(handle)
            _lib = handle
        return _lib


def check(status: int) -> None:
    if status != 0:
        msg = lib().p2bw_last_error().decode("utf-8", "replace")
        raise P2bwError(msg)


def call(name: str, *args) -> None:
    check(getattr(lib(), name)(*args))
