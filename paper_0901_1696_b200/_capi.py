"""ctypes binding of the C ABI in ``include/rfpk_b200.h`` (librfpk_b200.so).

There is no fallback: if the shared library is missing or no CUDA device is
present, :func:`lib` raises, so nothing in the package silently computes on
the CPU.
"""

from __future__ import annotations

import ctypes
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("RFPK_LIB") or os.path.join(_HERE, "librfpk_b200.so")

_c = ctypes.c_char
_i64 = ctypes.c_int64
_d = ctypes.c_double
_p = ctypes.c_void_p
_int = ctypes.c_int

# symbol -> argument types (mirrors include/rfpk_b200.h; the stream is last)
_MAT = [_p, _i64, _i64, _i64, _i64]
SIGNATURES = {
    "rfpk_version": ([], ctypes.c_char_p),
    "rfpk_device_sms": ([], _int),
    "rfpk_launch_count": ([], ctypes.c_longlong),
    "rfpk_graph_cache_clear": ([], _int),
    "rfpk_dtrttf": ([_c, _c, _i64, _p, _i64, _p, _p], _int),
    "rfpk_ztrttf": ([_c, _c, _i64, _p, _i64, _p, _p], _int),
    "rfpk_dtfttr": ([_c, _c, _i64, _p, _p, _i64, _p], _int),
    "rfpk_ztfttr": ([_c, _c, _i64, _p, _p, _i64, _p], _int),
    "rfpk_dtpttf": ([_c, _c, _i64, _p, _p, _p], _int),
    "rfpk_ztpttf": ([_c, _c, _i64, _p, _p, _p], _int),
    "rfpk_dtfttp": ([_c, _c, _i64, _p, _p, _p], _int),
    "rfpk_ztfttp": ([_c, _c, _i64, _p, _p, _p], _int),
    "rfpk_dtrttp": ([_c, _i64, _p, _i64, _p, _p], _int),
    "rfpk_ztrttp": ([_c, _i64, _p, _i64, _p, _p], _int),
    "rfpk_dtpttr": ([_c, _i64, _p, _p, _i64, _p], _int),
    "rfpk_ztpttr": ([_c, _i64, _p, _p, _i64, _p], _int),
    "rfpk_dpftrf": ([_c, _c, _i64, _p, _p, _p], _int),
    "rfpk_zpftrf": ([_c, _c, _i64, _p, _p, _p], _int),
    "rfpk_dpftrs": ([_c, _c, _i64, _i64, _p, _p, _i64, _p, _p], _int),
    "rfpk_zpftrs": ([_c, _c, _i64, _i64, _p, _p, _i64, _p, _p], _int),
    "rfpk_dpftrs_ex": ([_c, _c, _i64, _i64, _p, _p, _i64, _i64, _p, _p], _int),
    "rfpk_zpftrs_ex": ([_c, _c, _i64, _i64, _p, _p, _i64, _i64, _p, _p], _int),
    "rfpk_dtftri": ([_c, _c, _c, _i64, _p, _p, _p], _int),
    "rfpk_ztftri": ([_c, _c, _c, _i64, _p, _p, _p], _int),
    "rfpk_dpftri": ([_c, _c, _i64, _p, _p, _p], _int),
    "rfpk_zpftri": ([_c, _c, _i64, _p, _p, _p], _int),
    "rfpk_dpftrf_host": ([_c, _c, _i64, _p, _p, _p, _p], _int),
    "rfpk_zpftrf_host": ([_c, _c, _i64, _p, _p, _p, _p], _int),
    "rfpk_dpfsv": ([_c, _c, _i64, _i64, _p, _p, _i64, _p, _p], _int),
    "rfpk_zpfsv": ([_c, _c, _i64, _i64, _p, _p, _i64, _p, _p], _int),
    "rfpk_dpfsv_host": ([_c, _c, _i64, _i64, _p, _p, _p, _p, _p, _i64, _p, _p], _int),
    "rfpk_zpfsv_host": ([_c, _c, _i64, _i64, _p, _p, _p, _p, _p, _i64, _p, _p], _int),
    "rfpk_phase_clock": ([_int], _int),
    "rfpk_phase_time": ([ctypes.c_char_p, _p, _p], _int),
    "rfpk_dpptrf": ([_c, _i64, _p, _p, _p], _int),
    "rfpk_zpptrf": ([_c, _i64, _p, _p, _p], _int),
    "rfpk_dpptrs": ([_c, _i64, _i64, _p, _p, _i64, _i64, _p, _p], _int),
    "rfpk_zpptrs": ([_c, _i64, _i64, _p, _p, _i64, _i64, _p, _p], _int),
    "rfpk_dtfsm": ([_c, _c, _c, _c, _c, _i64, _i64, _d, _p, _p, _i64, _i64, _p, _p], _int),
    "rfpk_ztfsm": ([_c, _c, _c, _c, _c, _i64, _i64, _d, _d, _p, _p, _i64, _i64, _p, _p], _int),
    "rfpk_dsfrk": ([_c, _c, _c, _i64, _i64, _d, _p, _i64, _i64, _d, _p, _p], _int),
    "rfpk_zhfrk": ([_c, _c, _c, _i64, _i64, _d, _p, _i64, _i64, _d, _p, _int, _p], _int),
    "rfpk_dlansf": ([_c, _c, _c, _i64, _p, _p, _p], _int),
    "rfpk_zlansf": ([_c, _c, _c, _i64, _p, _p, _p], _int),
    "rfpk_dpftrf_batched": ([_c, _c, _i64, _p, _i64, _i64, _p, _p], _int),
    "rfpk_dpftrs_batched": ([_c, _c, _i64, _i64, _p, _i64, _p, _i64, _i64, _i64, _p, _p], _int),
    "rfpk_dpftrf_pftrs_batched": ([_c, _c, _i64, _i64, _p, _i64, _p, _i64, _i64, _i64, _p, _p],
                                  _int),
    "rfpk_dgemm": ([_c, _c, _d] + _MAT + _MAT + [_d] + _MAT + [_p], _int),
    "rfpk_zgemm": ([_c, _c, _d, _d] + _MAT + _MAT + [_d, _d] + _MAT + [_p], _int),
    "rfpk_dtrsm": ([_c, _c, _c, _c, _d, _p, _i64, _i64, _i64] + _MAT + [_p, _p], _int),
    "rfpk_ztrsm": ([_c, _c, _c, _c, _d, _d, _p, _i64, _i64, _i64] + _MAT + [_p, _p], _int),
    "rfpk_dtrmm": ([_c, _c, _c, _c, _d, _p, _i64, _i64, _i64] + _MAT + [_p], _int),
    "rfpk_ztrmm": ([_c, _c, _c, _c, _d, _d, _p, _i64, _i64, _i64] + _MAT + [_p], _int),
    "rfpk_dsyrk": ([_c, _c, _d] + _MAT + [_d, _p, _i64, _i64, _i64, _p], _int),
    "rfpk_zsyrk": ([_c, _c, _d] + _MAT + [_d, _p, _i64, _i64, _i64, _int, _p], _int),
    "rfpk_dpotrf": ([_c, _p, _i64, _i64, _i64, _p, _p], _int),
    "rfpk_zpotrf": ([_c, _p, _i64, _i64, _i64, _p, _p], _int),
    "rfpk_dtrtri": ([_c, _c, _p, _i64, _i64, _i64, _p, _p], _int),
    "rfpk_ztrtri": ([_c, _c, _p, _i64, _i64, _i64, _p, _p], _int),
    "rfpk_dlauum": ([_c, _p, _i64, _i64, _i64, _p], _int),
    "rfpk_zlauum": ([_c, _p, _i64, _i64, _i64, _p], _int),
}

_LIB = None


def load_library(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load the shared library and declare every exported signature.  Works
    without a GPU (no CUDA call is made)."""
    global _LIB
    if _LIB is None:
        if not os.path.exists(path):
            raise ImportError(
                f"librfpk_b200.so not found at {path}; build it with "
                "`python -c 'import __graft_entry__ as g; g.build()'` (no CPU fallback exists)")
        lib = ctypes.CDLL(path)
        for name, (argtypes, restype) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.argtypes = argtypes
            fn.restype = restype
        _LIB = lib
    return _LIB


def lib() -> ctypes.CDLL:
    """The library, after checking that a CUDA device is usable."""
    if not torch.cuda.is_available():
        raise RuntimeError("paper_0901_1696_b200 requires a CUDA device (B200, sm_100a); "
                           "there is no CPU fallback")
    return load_library()


def stream_handle(device=None) -> int:
    return torch.cuda.current_stream(device).cuda_stream


def flag(ch: str) -> bytes:
    return ch.encode("ascii")


def check(rc: int, fn: str) -> None:
    if rc < 0:
        raise ValueError(f"{fn}: illegal value of argument {-rc}")
    if rc > 0:
        raise RuntimeError(f"{fn}: CUDA error {rc}")
