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
    ]


class Op(C.Structure):
    _fields_ = [("kind", C.c_int), ("microbatch", C.c_int), ("weight_version", C.c_int)]


def _declare(lib: C.CDLL) -> None:
    i, ll, vp, f, d = C.c_int, C.c_longlong, C.c_void_p, C.c_float, C.c_double
    lib.p2bw_last_error.restype = C.c_char_p
    lib.p2bw_version.restype = C.c_char_p
    lib.p2bw_kernel_gemm_bf16.argtypes = [vp, ll, i, vp, ll, i, i, i, i, C.POINTER(GemmEpilogue), vp]


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
