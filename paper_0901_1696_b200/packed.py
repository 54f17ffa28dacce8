"""Full <-> column-packed conversions on the device (packed.py:41-67 of the
reference).  ``pack``/``unpack`` are the plumbing that produces the packed
input of BASELINE config 2's packed round trip; each is one launch of the
tiled copy kernel (C ABI ``rfpk_?trttp`` / ``rfpk_?tpttr``).

The reference's Level-2 packed Cholesky (``pptrf_ref``/``pptrs_ref``) and
SPD generator are comparators outside the RFPF hot path (SURVEY 2, rows
5b/5c) and are not rebuilt here.
"""

from __future__ import annotations

import torch

from . import _capi
from .convert import PackedTriangle, _call, _colmajor, _ld, _prefix, as_device

__all__ = ["pack", "unpack"]


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
