"""RFP / packed containers and the full <-> packed <-> RFP conversions, on
B200 device memory.

Drop-in for the reference ``rfpk.convert`` (convert.py): same class and
function names, argument order, return types, error types and messages.
Buffers are ``torch.Tensor`` on the current CUDA device (float64 or
complex128).  NumPy arrays / CPU tensors passed in are copied to the device
(a convenience the reference did not need); results are always device
tensors.  Every conversion is one launch of the tiled copy kernel in
``csrc/rfp.cu`` through the C ABI -- there is no host-side data movement and
no CPU fallback.

Reference map: FactorState convert.py:28-34; RfpTriangle :46-95;
PackedTriangle :98-139; trttf :156-186; tfttr :189-217; tpttf :220-246;
tfttp :249-275.
"""

from __future__ import annotations

import enum

import numpy as np
import torch

from . import _capi
from .layout import LayoutDescriptor, make_descriptor, normalize_flag

__all__ = [
    "FactorState",
    "RfpTriangle",
    "PackedTriangle",
    "trttf",
    "tfttr",
    "tpttf",
    "tfttp",
    "as_device",
]


class FactorState(enum.Enum):
    """Lifecycle of an :class:`RfpTriangle`'s values (convert.py:28-34)."""

    UNFACTORED = "unfactored"
    CHOLESKY = "cholesky"
    TRIANGULAR_INVERSE = "triangular_inverse"
    FULL_INVERSE = "full_inverse"


def as_device(x, device=None) -> torch.Tensor:
    """Float64/complex128 CUDA tensor view of ``x`` (copies only when the
    dtype or device differs; mirrors convert.py:37-43 dtype coercion)."""
    if not isinstance(x, torch.Tensor):
        x = torch.from_numpy(np.ascontiguousarray(np.asarray(x)) if not isinstance(x, np.ndarray)
                             else x)
    if x.dtype not in (torch.float64, torch.complex128):
        x = x.to(torch.complex128 if x.is_complex() else torch.float64)
    if not x.is_cuda:
        _capi.lib()  # raises without a device: no CPU fallback
        x = x.to(device or torch.device("cuda", torch.cuda.current_device()))
    return x


def _colmajor(a: torch.Tensor) -> torch.Tensor:
    """``a`` itself if column-major (unit row stride), else a column-major copy."""
    if a.stride(0) == 1 or a.shape[0] <= 1:
        return a
    return a.t().contiguous().t()


def _ld(a: torch.Tensor) -> int:
    return max(a.stride(1) if a.shape[1] > 1 else a.shape[0], a.shape[0], 1)


def _prefix(dtype) -> str:
    return "z" if dtype == torch.complex128 else "d"


class RfpTriangle:
    """Minimal-storage buffer of ``n(n+1)/2`` scalars in RFP layout
    (convert.py:46-95).  ``data`` is a 1-D CUDA tensor."""

    __slots__ = ("data", "desc", "state")

    def __init__(self, data, desc: LayoutDescriptor, state: FactorState = FactorState.UNFACTORED):
        data = as_device(data)
        if data.dim() != 1 or not data.is_contiguous():
            data = data.reshape(-1).contiguous()
        if data.shape[0] != desc.nt:
            raise ValueError(f"buffer length {data.shape[0]} != nt={desc.nt} for n={desc.n}")
        self.data = data
        self.desc = desc
        self.state = state

    @classmethod
    def zeros(cls, n: int, uplo: str, transr: str, dtype=torch.float64) -> "RfpTriangle":
        desc = make_descriptor(n, uplo, transr)
        dtype = _torch_dtype(dtype)
        _capi.lib()
        return cls(torch.zeros(desc.nt, dtype=dtype, device="cuda"), desc)

    @property
    def dtype(self):
        return self.data.dtype

    def rect(self) -> torch.Tensor:
        """Stored rectangle (``ldar x n1``, or ``n1 x ldar`` for 'T'), no copy."""
        d = self.desc
        if d.transr == "N":
            return self.data.view(d.n1, d.ldar).t()
        return self.data.view(d.ldar, d.n1).t()

    def rect_normal(self) -> torch.Tensor:
        """The ``ldar x n1`` rectangle regardless of transr (a view)."""
        r = self.rect()
        return r if self.desc.transr == "N" else r.t()

    def copy(self) -> "RfpTriangle":
        return RfpTriangle(self.data.clone(), self.desc, self.state)

    def __repr__(self):
        d = self.desc
        return (f"RfpTriangle(n={d.n}, uplo={d.uplo!r}, transr={d.transr!r}, "
                f"state={self.state.value}, dtype={self.dtype})")


class PackedTriangle:
    """LAPACK column-packed triangle (convert.py:98-139)."""

    __slots__ = ("data", "n", "uplo")

    def __init__(self, data, n: int, uplo: str):
        data = as_device(data)
        if data.dim() != 1 or not data.is_contiguous():
            data = data.reshape(-1).contiguous()
        if data.shape[0] != n * (n + 1) // 2:
            raise ValueError(f"packed length {data.shape[0]} != {n * (n + 1) // 2} for n={n}")
        u = str(uplo).upper()[:1]
        if u not in ("L", "U"):
            raise ValueError(f"uplo must be 'L' or 'U', got {u!r}")
        self.data = data
        self.n = int(n)
        self.uplo = u

    @classmethod
    def zeros(cls, n: int, uplo: str, dtype=torch.float64) -> "PackedTriangle":
        _capi.lib()
        return cls(torch.zeros(n * (n + 1) // 2, dtype=_torch_dtype(dtype), device="cuda"), n, uplo)

    @property
    def dtype(self):
        return self.data.dtype

    def copy(self) -> "PackedTriangle":
        return PackedTriangle(self.data.clone(), self.n, self.uplo)

    def column(self, j: int) -> torch.Tensor:
        """View of packed column ``j`` (rows j..n-1 lower, 0..j upper)."""
        n = self.n
        if self.uplo == "L":
            off = j * n - j * (j - 1) // 2
            return self.data[off:off + n - j]
        off = j * (j + 1) // 2
        return self.data[off:off + j + 1]

    def __repr__(self):
        return f"PackedTriangle(n={self.n}, uplo={self.uplo!r}, dtype={self.dtype})"


def _torch_dtype(dtype):
    if dtype in (torch.float64, torch.complex128):
        return dtype
    return torch.complex128 if np.dtype(dtype).kind == "c" else torch.float64


def _call(name: str, *args) -> None:
    fn = getattr(_capi.lib(), name)
    _capi.check(fn(*args), name)


def trttf(a, uplo: str, transr: str) -> RfpTriangle:
    """Declared triangle of the full ``(ld, n)`` matrix ``a`` -> new RFP
    buffer (convert.py:156-186); only ``a[:n, :n]``'s triangle is read."""
    a = as_device(a)
    if a.dim() != 2:
        raise ValueError("full input must be 2-dimensional")
    n = a.shape[1]
    if a.shape[0] < n:
        raise ValueError(f"leading dimension {a.shape[0]} < n={n}")
    desc = make_descriptor(n, uplo, transr)
    out = torch.empty(desc.nt, dtype=a.dtype, device=a.device)
    if n:
        a = _colmajor(a)
        _call(f"rfpk_{_prefix(a.dtype)}trttf", _capi.flag(desc.transr), _capi.flag(desc.uplo), n,
              a.data_ptr(), _ld(a), out.data_ptr(), _capi.stream_handle(a.device))
    return RfpTriangle(out, desc)


def tfttr(r: RfpTriangle, ld=None) -> torch.Tensor:
    """RFP -> new column-major ``(ld, n)`` tensor, zero outside the triangle
    (convert.py:189-217)."""
    desc = r.desc
    n = desc.n
    ld = n if ld is None else int(ld)
    if ld < n:
        raise ValueError(f"leading dimension {ld} < n={n}")
    out = torch.empty((n, ld), dtype=r.dtype, device=r.data.device).t()
    if n == 0:
        return out.zero_()
    _call(f"rfpk_{_prefix(r.dtype)}tfttr", _capi.flag(desc.transr), _capi.flag(desc.uplo), n,
          r.data.data_ptr(), out.data_ptr(), max(ld, 1), _capi.stream_handle(r.data.device))
    return out


def tpttf(p: PackedTriangle, transr: str) -> RfpTriangle:
    """Column-packed triangle -> new RFP buffer (convert.py:220-246)."""
    desc = make_descriptor(p.n, p.uplo, transr)
    out = torch.empty(desc.nt, dtype=p.dtype, device=p.data.device)
    if p.n:
        _call(f"rfpk_{_prefix(p.dtype)}tpttf", _capi.flag(desc.transr), _capi.flag(desc.uplo),
              p.n, p.data.data_ptr(), out.data_ptr(), _capi.stream_handle(p.data.device))
    return RfpTriangle(out, desc)


def tfttp(r: RfpTriangle) -> PackedTriangle:
    """RFP -> new column-packed triangle (convert.py:249-275)."""
    desc = r.desc
    out = torch.empty(desc.nt, dtype=r.dtype, device=r.data.device)
    if desc.n:
        _call(f"rfpk_{_prefix(r.dtype)}tfttp", _capi.flag(desc.transr), _capi.flag(desc.uplo),
              desc.n, r.data.data_ptr(), out.data_ptr(), _capi.stream_handle(r.data.device))
    return PackedTriangle(out, desc.n, desc.uplo)


def _uplo(u) -> str:
    return normalize_flag(u, "LU", "uplo")
