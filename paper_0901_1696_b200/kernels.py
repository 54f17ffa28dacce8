"""Full-format dense kernels on device views (the reference ``rfpk.kernels``,
kernels.py:91-606), as sm_100a kernels behind the C ABI.

Each function works in place on 2-D CUDA tensors (any view whose row or
column stride is 1 -- transposed views included, exactly how the reference
addresses T1/T2/S1).  Flag parsing, shape checks, messages and the
``SingularMatrixError`` contract follow the reference.  ``nb`` is accepted
for signature compatibility; the device kernels use compile-time tiles.
"""

from __future__ import annotations

import os

import numpy as np
import torch

from . import _capi
from .convert import _prefix, as_device

__all__ = [
    "SingularMatrixError",
    "default_block_size",
    "gemm",
    "trsm",
    "trmm",
    "syrk_herk",
    "potrf_ref",
    "trtri_ref",
    "lauum_ref",
]

_DEFAULT_NB = max(1, int(os.environ.get("RFPK_NB", "64")))


class SingularMatrixError(np.linalg.LinAlgError):
    """Zero diagonal entry in a non-unit triangular matrix (kernels.py:38-46);
    ``index`` is 1-based."""

    def __init__(self, index: int):
        self.index = int(index)
        super().__init__(f"zero diagonal entry at position {self.index}")


def default_block_size() -> int:
    return _DEFAULT_NB


def _check(flag, allowed: str, what: str) -> str:
    f = str(flag).upper()[:1]
    if f not in allowed:
        raise ValueError(f"{what} must be one of {tuple(allowed)}, got {flag!r}")
    return f


def _mat(a, what: str) -> torch.Tensor:
    if not isinstance(a, torch.Tensor):
        a = as_device(a)
    if a.dim() != 2:
        raise ValueError(f"{what} must be 2-dimensional, got ndim={a.dim()}")
    if not a.is_cuda:
        raise ValueError(f"{what} must be a CUDA tensor (in-place device kernel)")
    return a


def _square(a, what: str) -> torch.Tensor:
    a = _mat(a, what)
    if a.shape[0] != a.shape[1]:
        raise ValueError(f"{what} must be square, got shape {tuple(a.shape)}")
    return a


class _Unit:
    """A view with a unit stride (the tensor itself, or a column-major
    working copy that is written back on exit)."""

    def __init__(self, t: torch.Tensor, writeback: bool):
        self.orig = t
        ok = t.stride(0) == 1 or t.stride(1) == 1 or t.shape[0] <= 1 or t.shape[1] <= 1
        self.t = t if ok else t.t().contiguous().t()
        self.writeback = writeback and self.t is not t

    def args(self):
        t = self.t
        return (t.data_ptr(), t.shape[0], t.shape[1], t.stride(0), t.stride(1))

    def done(self):
        if self.writeback:
            self.orig.copy_(self.t)


def _same_dtype(*ts):
    cplx = any(t.is_complex() for t in ts)
    dt = torch.complex128 if cplx else torch.float64
    for t in ts:
        if t.dtype != dt:
            raise ValueError(f"all operands must be {dt}, got {t.dtype}")
    return dt


def _run(name, *args):
    _capi.check(getattr(_capi.lib(), name)(*args), name)


def _cz(v):
    v = complex(v)
    return (v.real, v.imag)


def gemm(transa: str, transb: str, alpha, a, b, beta, c) -> None:
    """``C <- alpha*op(A)@op(B) + beta*C`` in place on ``c`` (kernels.py:129-145)."""
    transa = _check(transa, "NTC", "transa")
    transb = _check(transb, "NTC", "transb")
    a, b, c = _mat(a, "a"), _mat(b, "b"), _mat(c, "c")
    m, n = c.shape
    if alpha != 0:
        sa = tuple(a.shape) if transa == "N" else tuple(a.shape)[::-1]
        sb = tuple(b.shape) if transb == "N" else tuple(b.shape)[::-1]
        if sa[0] != m or sb[1] != n or sa[1] != sb[0]:
            raise ValueError(f"gemm shape mismatch: op(a)={sa}, op(b)={sb}, c={tuple(c.shape)}")
    dt = _same_dtype(a, b, c)
    ua, ub, uc = _Unit(a, False), _Unit(b, False), _Unit(c, True)
    st = _capi.stream_handle(c.device)
    if dt == torch.complex128:
        _run("rfpk_zgemm", _capi.flag(transa), _capi.flag(transb), *_cz(alpha), *ua.args(),
             *ub.args(), *_cz(beta), *uc.args(), st)
    else:
        _run("rfpk_dgemm", _capi.flag(transa), _capi.flag(transb), float(alpha), *ua.args(),
             *ub.args(), float(beta), *uc.args(), st)
    uc.done()


def _tri(name, side, uplo, trans, diag, alpha, a, b, with_info):
    side = _check(side, "LR", "side")
    uplo = _check(uplo, "LU", "uplo")
    trans = _check(trans, "NTC", "trans")
    diag = _check(diag, "NU", "diag")
    a, b = _square(a, "a"), _mat(b, "b")
    k = b.shape[0] if side == "L" else b.shape[1]
    if a.shape[0] != k:
        raise ValueError(f"{name} shape mismatch: a={tuple(a.shape)}, b={tuple(b.shape)}")
    if b.numel() == 0 or k == 0:
        return
    dt = _same_dtype(a, b) if a.is_complex() or not b.is_complex() else None
    if dt is None:  # real triangle, complex B: promote the triangle
        a = a.to(torch.complex128)
        dt = torch.complex128
    ua, ub = _Unit(a, False), _Unit(b, True)
    pa = ua.args()
    tri_a = (pa[0], pa[1], pa[3], pa[4])
    flags = (_capi.flag(side), _capi.flag(uplo), _capi.flag(trans), _capi.flag(diag))
    st = _capi.stream_handle(b.device)
    info = torch.zeros(1, dtype=torch.int32, device=b.device) if with_info else None
    extra = (info.data_ptr(), st) if with_info else (st,)
    if dt == torch.complex128:
        _run(f"rfpk_z{name}", *flags, *_cz(alpha), *tri_a, *ub.args(), *extra)
    else:
        _run(f"rfpk_d{name}", *flags, float(alpha), *tri_a, *ub.args(), *extra)
    if with_info:
        v = int(info.item())
        if v:
            raise SingularMatrixError(v)
    ub.done()


def trsm(side: str, uplo: str, trans: str, diag: str, alpha, a, b, nb=None) -> None:
    """Solve ``op(A) X = alpha B`` (side 'L') or ``X op(A) = alpha B`` (side
    'R') in place on ``b`` (kernels.py:218-238); a zero diagonal (diag 'N')
    raises :class:`SingularMatrixError` with its 1-based index."""
    _tri("trsm", side, uplo, trans, diag, alpha, a, b, True)


def trmm(side: str, uplo: str, trans: str, diag: str, alpha, a, b, nb=None) -> None:
    """``B <- alpha op(A) B`` / ``alpha B op(A)`` in place (kernels.py:307-321)."""
    _tri("trmm", side, uplo, trans, diag, alpha, a, b, False)


def syrk_herk(uplo: str, trans: str, alpha, a, beta, c, hermitian: bool = False) -> None:
    """Rank-k update of the declared triangle of ``c`` (kernels.py:405-423)."""
    uplo = _check(uplo, "LU", "uplo")
    trans = _check(trans, "NTC", "trans")
    a, c = _mat(a, "a"), _square(c, "c")
    alpha, beta = float(alpha), float(beta)
    n = c.shape[0]
    rows = a.shape[0] if trans == "N" else a.shape[1]
    if alpha != 0 and rows != n:
        raise ValueError(f"syrk_herk shape mismatch: a={tuple(a.shape)}, c={tuple(c.shape)}")
    dt = _same_dtype(a, c)
    ua, uc = _Unit(a, False), _Unit(c, True)
    pc = uc.args()
    st = _capi.stream_handle(c.device)
    if dt == torch.complex128:
        _run("rfpk_zsyrk", _capi.flag(uplo), _capi.flag(trans), alpha, *ua.args(), beta, pc[0],
             pc[1], pc[3], pc[4], 1 if hermitian else 0, st)
    else:
        _run("rfpk_dsyrk", _capi.flag(uplo), _capi.flag(trans), alpha, *ua.args(), beta, pc[0],
             pc[1], pc[3], pc[4], st)
    uc.done()


def _square_call(prefix_name, a, *flags, with_info=True):
    ua = _Unit(a, True)
    p = ua.args()
    st = _capi.stream_handle(a.device)
    info = torch.zeros(1, dtype=torch.int32, device=a.device)
    name = f"rfpk_{_prefix(a.dtype)}{prefix_name}"
    if with_info:
        _run(name, *flags, p[0], p[1], p[3], p[4], info.data_ptr(), st)
    else:
        _run(name, *flags, p[0], p[1], p[3], p[4], st)
    v = int(info.item()) if with_info else 0
    ua.done()
    return v


def potrf_ref(uplo: str, a, nb=None) -> int:
    """Cholesky in place: ``L L^H`` ('L') / ``U^H U`` ('U'); returns 0 or
    the 1-based first non-positive leading minor (kernels.py:468-496)."""
    uplo = _check(uplo, "LU", "uplo")
    a = _square(a, "a")
    if a.shape[0] == 0:
        return 0
    _same_dtype(a)
    return _square_call("potrf", a, _capi.flag(uplo))


def trtri_ref(uplo: str, diag: str, a, nb=None) -> int:
    """Triangular inverse in place; 0 or the 1-based index of a zero
    diagonal, matrix untouched on failure (kernels.py:515-547)."""
    uplo = _check(uplo, "LU", "uplo")
    diag = _check(diag, "NU", "diag")
    a = _square(a, "a")
    if a.shape[0] == 0:
        return 0
    _same_dtype(a)
    return _square_call("trtri", a, _capi.flag(uplo), _capi.flag(diag))


def lauum_ref(uplo: str, a, nb=None) -> None:
    """``A <- U U^H`` ('U') / ``L^H L`` ('L') in place (kernels.py:575-606)."""
    uplo = _check(uplo, "LU", "uplo")
    a = _square(a, "a")
    if a.shape[0] == 0:
        return
    _same_dtype(a)
    _square_call("lauum", a, _capi.flag(uplo), with_info=False)
