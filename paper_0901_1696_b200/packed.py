"""Full <-> column-packed conversions on the device (packed.py:41-67 of the
reference).  ``pack``/``unpack`` are the plumbing that produces the packed
input of BASELINE config 2's packed round trip; each is one launch of the
tiled copy kernel (C ABI ``rfpk_?trttp`` / ``rfpk_?tpttr``).

``pptrf_ref``/``pptrs_ref`` are the reference's Level-2 packed Cholesky
comparator (packed.py:70-146).  Here they keep the
reference's names, arguments, return values and errors, but compute through
RFP on the device (C ABI ``rfpk_?pptrf`` / ``rfpk_?pptrs``: packed -> RFP ->
pftrf/pftrs -> packed), so the packed path runs on the same tensor-core
kernels.  The SPD generator (``spd_generate``) stays out of scope.
"""

from __future__ import annotations

import torch

from . import _capi
from .convert import PackedTriangle, _call, _colmajor, _ld, _prefix, as_device
from .rfp import _info, _rhs_view

__all__ = ["pack", "unpack", "pptrf_ref", "pptrs_ref"]


def pack(a, uplo: str) -> PackedTriangle:
    """Column-pack the declared triangle of the full matrix ``a``."""
    a = as_device(a)
    if a.dim() != 2:
        raise ValueError("full input must be 2-dimensional")
    n = a.shape[1]
    if a.shape[0] < n:
        raise ValueError(f"leading dimension {a.shape[0]} < n={n}")
    u = str(uplo).upper()[:1]
    if u not in ("L", "U"):
        raise ValueError(f"uplo must be 'L' or 'U', got {uplo!r}")
    out = torch.empty(n * (n + 1) // 2, dtype=a.dtype, device=a.device)
    if n:
        a = _colmajor(a)
        _call(f"rfpk_{_prefix(a.dtype)}trttp", _capi.flag(u), n, a.data_ptr(), _ld(a),
              out.data_ptr(), _capi.stream_handle(a.device))
    return PackedTriangle(out, n, u)


def unpack(p: PackedTriangle, ld=None) -> torch.Tensor:
    """Expand a packed triangle to a column-major ``(ld, n)`` tensor with
    zeros outside the triangle."""
    n = p.n
    ld = n if ld is None else int(ld)
    if ld < n:
        raise ValueError(f"leading dimension {ld} < n={n}")
    out = torch.empty((n, ld), dtype=p.dtype, device=p.data.device).t()
    if n == 0:
        return out.zero_()
    _call(f"rfpk_{_prefix(p.dtype)}tpttr", _capi.flag(p.uplo), n, p.data.data_ptr(),
          out.data_ptr(), max(ld, 1), _capi.stream_handle(p.data.device))
    return out


def pptrf_ref(p: PackedTriangle) -> int:
    """Packed Cholesky factorization, in place (packed.py:70-108).  Returns 0
    or the 1-based order of the first non-positive leading minor."""
    if p.n == 0:
        return 0
    info = _info(p.data.device)
    _call(f"rfpk_{_prefix(p.dtype)}pptrf", _capi.flag(p.uplo), p.n, p.data.data_ptr(),
          info.data_ptr(), _capi.stream_handle(p.data.device))
    return int(info.item())


class _PackedOrder:
    """The two attributes of an RfpTriangle that ``rfp._rhs_view`` reads."""

    def __init__(self, p: PackedTriangle):
        self.desc = type("D", (), {"n": p.n})()
        self.dtype = p.dtype


def pptrs_ref(p: PackedTriangle, b) -> None:
    """Solve ``A @ X = B`` in place from a packed Cholesky factor
    (packed.py:111-146); ``b`` is (n,) or (n, nrhs), device or host."""
    bv, foreign = _rhs_view(_PackedOrder(p), b)
    if p.n == 0 or bv.shape[1] == 0:
        return
    work = bv
    data = p.data
    if bv.dtype not in (torch.float64, torch.complex128) or (bv.stride(0) != 1 and bv.stride(1) != 1):
        work = bv.to(torch.complex128 if bv.is_complex() else torch.float64).t().contiguous().t()
    if work.is_complex() and not data.is_complex():
        data = data.to(torch.complex128)
    info = _info(work.device)
    _call(f"rfpk_{_prefix(data.dtype)}pptrs", _capi.flag(p.uplo), p.n, work.shape[1],
          data.data_ptr(), work.data_ptr(), work.stride(0), work.stride(1), info.data_ptr(),
          _capi.stream_handle(work.device))
    if work is not bv:
        bv.copy_(work)
    if foreign is not None:
        host = bv.reshape(tuple(foreign.shape)).cpu()
        if isinstance(foreign, torch.Tensor):
            foreign.copy_(host)
        else:
            foreign[...] = host.numpy()
