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
    "rfpk_set_tuning": ([ctypes.c_char_p, ctypes.c_longlong], _int),
    "rfpk_get_tuning": ([ctypes.c_char_p, _p], _int),
    "rfpk_reset_tuning": ([], _int),
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
    "rfpk_phase_labels": ([_p, _i64], _i64),
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


class phase_clock:
    """Context manager around the library's phase clock (rfpk_phase_clock):
    CUDA event pairs on the launching streams around every SRPA step and
    every library kernel launch (direct calls; graph replays are not
    traced).  ``table()`` -> {label: (total_ms, count)} after the block."""

    def __enter__(self):
        load_library().rfpk_phase_clock(1)
        self._table = None
        return self

    def __exit__(self, *exc):
        self._table = self.table()
        load_library().rfpk_phase_clock(0)
        return False

    def table(self):
        if self._table is not None:
            return self._table
        lib = load_library()
        need = lib.rfpk_phase_labels(None, 0)
        buf = ctypes.create_string_buffer(int(need))
        lib.rfpk_phase_labels(buf, need)
        out = {}
        for lab in buf.value.decode().splitlines():
            ms, cnt = ctypes.c_double(0.0), ctypes.c_int64(0)
            lib.rfpk_phase_time(lab.encode(), ctypes.byref(ms), ctypes.byref(cnt))
            out[lab] = (float(ms.value), int(cnt.value))
        return out


TUNING_DEFAULTS = {"oop_max": 4096, "t2_copy_min": 2048, "panel_max": 4096,
                   "pfsv_overlap_min": 512, "overlap": 1, "graphs": 1, "graph_max_n": 8192,
                   "gemm_wide": 0, "batched_generic": 0, "trace": 0, "trsm_split": 1,
                   "zpotrf_split_min": 9000}


def set_tuning(name: str, value: int) -> None:
    """Set one of the library's path thresholds (rfpk_set_tuning; see
    include/rfpk_b200.h).  Drops every cached CUDA graph."""
    if load_library().rfpk_set_tuning(name.encode(), int(value)) != 0:
        raise KeyError(f"unknown tuning knob {name!r}")


def get_tuning(name: str) -> int:
    v = ctypes.c_longlong(0)
    if load_library().rfpk_get_tuning(name.encode(), ctypes.byref(v)) != 0:
        raise KeyError(f"unknown tuning knob {name!r}")
    return int(v.value)


class tuning:
    """Context manager: ``with tuning(panel_max=256): ...`` sets knobs and
    restores their previous values on exit."""

    def __init__(self, **knobs):
        self.knobs = knobs
        self.saved = {}

    def __enter__(self):
        for k, v in self.knobs.items():
            self.saved[k] = get_tuning(k)
            set_tuning(k, v)
        return self

    def __exit__(self, *exc):
        for k, v in self.saved.items():
            set_tuning(k, v)
        return False


def flag(ch: str) -> bytes:
    return ch.encode("ascii")


def check(rc: int, fn: str) -> None:
    if rc < 0:
        raise ValueError(f"{fn}: illegal value of argument {-rc}")
    if rc > 0:
        raise RuntimeError(f"{fn}: CUDA error {rc}")
