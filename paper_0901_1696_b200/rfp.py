"""RFPF Cholesky factorization, solve and inversion on the B200.

Drop-in for the reference ``rfpk.rfp`` hot path (rfp.py:55-360): the same
entry points, argument order, return values, state machine and exceptions.
Each call is ONE call into the C ABI, which runs the whole SRPA chain
(potrf -> trsm -> syrk/herk -> potrf, etc.) as stream-ordered sm_100a
kernels on the RFP buffer in place; the Python layer only validates, then
reads the device ``info`` once (the reference's synchronous int return).

Extensions for BASELINE config 4: ``pftrf_batched`` / ``pftrs_batched`` /
``pftrf_pftrs_batched`` over many independent RFP buffers.
"""

from __future__ import annotations

import threading

import numpy as np
import torch

from . import _capi
from .convert import FactorState, RfpTriangle, _prefix, as_device
from .layout import make_descriptor, normalize_flag

__all__ = [
    "pftrf",
    "pftrf_from_host",
    "pfsv_from_host",
    "pfsv",
    "pftrs",
    "tfsm",
    "sfrk_hfrk",
    "tftri",
    "pftri",
    "lansf",
    "pftrf_batched",
    "pftrs_batched",
    "pftrf_pftrs_batched",
    "pftrf_pftrs_batched_from_host",
]


def _fn(name: str):
    return getattr(_capi.lib(), name)


def _run(name: str, *args) -> None:
    _capi.check(_fn(name)(*args), name)


_TLS = threading.local()


def _info(device) -> torch.Tensor:
    """A persistent per-thread, per-device info int: stable pointers let the
    C ABI's CUDA-graph cache replay repeated calls on the same buffers."""
    cache = getattr(_TLS, "info", None)
    if cache is None:
        cache = _TLS.info = {}
    dev = torch.device(device)
    idx = dev.index if dev.index is not None else torch.cuda.current_device()
    t = cache.get(idx)
    if t is None:
        t = cache[idx] = torch.zeros(1, dtype=torch.int32, device=torch.device("cuda", idx))
    return t


def pftrf(r: RfpTriangle) -> int:
    """Cholesky-factor the RFP-stored SPD/HPD matrix in place (rfp.py:55-91).

    Returns 0 (state -> CHOLESKY) or the 1-based order of the first
    non-positive leading minor (state unchanged)."""
    desc = r.desc
    if desc.n == 0:
        r.state = FactorState.CHOLESKY
        return 0
    info = _info(r.data.device)
    _run(f"rfpk_{_prefix(r.dtype)}pftrf", _capi.flag(desc.transr), _capi.flag(desc.uplo), desc.n,
         r.data.data_ptr(), info.data_ptr(), _capi.stream_handle(r.data.device))
    v = int(info.item())
    if v == 0:
        r.state = FactorState.CHOLESKY
    return v


def pfsv(r: RfpTriangle, b) -> int:
    """:func:`pftrf` then :func:`pftrs` on ``b`` in one call
    (rfp.py:55-136, the pair): the first solve with T1 and the S1 product run
    on the device concurrently with potrf(T2).  Returns pftrf's info; ``b``
    is solved in place only on success (0).  A device ``b`` that is not a
    column-major float64/complex128 (n, nrhs) view of the factor's dtype
    takes the two separate calls."""
    if r.state is not FactorState.UNFACTORED:
        raise ValueError(f"pfsv needs an unfactored matrix, state is {r.state.value}")
    desc = r.desc
    fast = (isinstance(b, torch.Tensor) and b.is_cuda and b.dim() == 2 and b.dtype == r.dtype
            and b.device == r.data.device and b.shape[0] == desc.n and b.stride(0) == 1
            and b.stride(1) >= max(desc.n, 1) and desc.n > 0)
    if not fast:
        v = pftrf(r)
        if v == 0:
            pftrs(r, b)
        return v
    keep = b.clone()
    info = _info(r.data.device)
    _run(f"rfpk_{_prefix(r.dtype)}pfsv", _capi.flag(desc.transr), _capi.flag(desc.uplo), desc.n,
         b.shape[1], r.data.data_ptr(), b.data_ptr(), b.stride(1), info.data_ptr(),
         _capi.stream_handle(r.data.device))
    v = int(info.item())
    if v == 0:
        r.state = FactorState.CHOLESKY
    else:
        b.copy_(keep)  # the reference's pftrs never runs after a failed pftrf
    return v


def pftrf_from_host(data, n: int, uplo: str, transr: str):
    """:func:`pftrf` of an RFP buffer that still sits in host memory, with
    the host->device transfer streamed under the factorization (the rows of
    T1/T2 first, S1's on a side stream, hidden by potrf(T1); C ABI
    ``rfpk_?pftrf_host``).  ``data``: CPU tensor (pinned for a truly
    asynchronous copy) or NumPy array of ``n(n+1)/2`` scalars.  Returns
    ``(RfpTriangle on the device, info)`` like ``pftrf``."""
    desc = make_descriptor(n, uplo, transr)
    host = data if isinstance(data, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(data))
    if host.is_cuda:
        raise ValueError("pftrf_from_host expects host memory; use pftrf for device buffers")
    if host.dtype not in (torch.float64, torch.complex128):
        host = host.to(torch.complex128 if host.is_complex() else torch.float64)
    host = host.reshape(-1).contiguous()
    if host.shape[0] != desc.nt:
        raise ValueError(f"buffer length {host.shape[0]} != nt={desc.nt} for n={desc.n}")
    _capi.lib()
    dev = torch.empty(desc.nt, dtype=host.dtype, device=torch.device("cuda", torch.cuda.current_device()))
    r = RfpTriangle(dev, desc)
    if desc.n == 0:
        r.state = FactorState.CHOLESKY
        return r, 0
    info = _info(dev.device)
    _run(f"rfpk_{_prefix(host.dtype)}pftrf_host", _capi.flag(desc.transr), _capi.flag(desc.uplo),
         desc.n, host.data_ptr(), dev.data_ptr(), info.data_ptr(), _capi.stream_handle(dev.device))
    v = int(info.item())
    if v == 0:
        r.state = FactorState.CHOLESKY
    return r, v


def pfsv_from_host(data, b, n: int, uplo: str, transr: str, out=None):
    """:func:`pftrf` then :func:`pftrs` for a problem that sits in host
    memory, with every transfer overlapped with the computation (C ABI
    ``rfpk_?pfsv_host``): the RFP buffer's T1/T2 rows first, its S1 rows and
    the right-hand side on a side stream under potrf(T1) and the S1 solve,
    and the solution's trailing block copied back during the last two solve
    steps.  ``data``: ``n(n+1)/2`` scalars, ``b``: (n,) or (n, nrhs) host
    arrays (pinned CPU tensors for truly asynchronous copies).  The solution
    is written into ``out`` (default: ``b``).  Returns ``(RfpTriangle on the
    device, info)`` like ``pftrf``; on failure the solution is unspecified."""
    desc = make_descriptor(n, uplo, transr)
    host = data if isinstance(data, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(data))
    bh = b if isinstance(b, torch.Tensor) else torch.from_numpy(np.asarray(b))
    if host.is_cuda or bh.is_cuda:
        raise ValueError("pfsv_from_host expects host memory; use pftrf/pftrs for device buffers")
    cplx = host.is_complex() or bh.is_complex()
    dt = torch.complex128 if cplx else torch.float64
    host = host.to(dt).reshape(-1).contiguous()
    if host.shape[0] != desc.nt:
        raise ValueError(f"buffer length {host.shape[0]} != nt={desc.nt} for n={desc.n}")
    flat = bh.dim() == 1
    b2 = bh.reshape(-1, 1) if flat else bh
    if b2.dim() != 2 or b2.shape[0] != n:
        raise ValueError(f"right-hand side shape {tuple(bh.shape)} does not match order {n}")
    bc = b2.to(dt)
    if not (bc.stride(0) == 1 and bc.stride(1) == max(n, 1)):
        bc = bc.t().contiguous().t()  # column-major, ld = n
    dst = out if out is not None else b

    def colmajor_view(t):
        """t as an (n, nrhs) column-major ld=n dt tensor sharing memory, or None"""
        if not isinstance(t, torch.Tensor) or t.is_cuda or t.dtype != dt:
            return None
        v = t.reshape(-1, 1) if t.dim() == 1 else t
        if v.shape != bc.shape or v.stride(0) != 1 or (v.shape[1] > 1 and v.stride(1) != max(n, 1)):
            return None
        return v

    xc = colmajor_view(dst)
    direct = xc is not None
    if not direct:
        xc = torch.empty((bc.shape[1], n), dtype=dt).t()
    _capi.lib()
    devn = torch.device("cuda", torch.cuda.current_device())
    d_arf = torch.empty(desc.nt, dtype=dt, device=devn)
    nrhs = bc.shape[1]
    d_b = torch.empty((nrhs, n), dtype=dt, device=devn).t()
    r = RfpTriangle(d_arf, desc)
    info = _info(devn)
    _run(f"rfpk_{_prefix(dt)}pfsv_host", _capi.flag(desc.transr), _capi.flag(desc.uplo), desc.n,
         nrhs, host.data_ptr(), d_arf.data_ptr(), bc.data_ptr(), d_b.data_ptr(), xc.data_ptr(),
         max(n, 1), info.data_ptr(), _capi.stream_handle(devn))
    v = int(info.item())  # synchronises: the solution is on the host
    if v == 0:
        r.state = FactorState.CHOLESKY
    if not direct:
        res = xc.reshape(bh.shape) if flat else xc
        if isinstance(dst, torch.Tensor):
            dst.copy_(res)
        else:
            dst[...] = res.numpy()
    return r, v


def _rhs_view(r: RfpTriangle, b):
    """(device 2-D view, host/foreign original or None, was_1d) (rfp.py:94-103)."""
    foreign = None
    if not isinstance(b, torch.Tensor) or not b.is_cuda:
        foreign = b
        bt = as_device(b)
    else:
        bt = b
    flat = bt.dim() == 1
    bv = bt.reshape(-1, 1) if flat else bt
    if bv.dim() != 2 or bv.shape[0] != r.desc.n:
        raise ValueError(
            f"right-hand side shape {tuple(bt.shape)} does not match order {r.desc.n}")
    if r.dtype == torch.complex128 and not bv.is_complex():
        raise ValueError("complex system needs a complex right-hand side")
    return bv, foreign


def pftrs(r: RfpTriangle, b) -> None:
    """Solve A X = B in place on ``b`` with the factor from :func:`pftrf`
    (rfp.py:106-136).  ``b`` is (n,) or (n, nrhs), any strides; a host
    (NumPy / CPU tensor) ``b`` is solved on the device and written back."""
    if r.state is not FactorState.CHOLESKY:
        raise ValueError(f"pftrs needs a Cholesky factor, state is {r.state.value}")
    bv, foreign = _rhs_view(r, b)
    desc = r.desc
    if desc.n == 0 or bv.shape[1] == 0:
        return
    work = bv
    data = r.data
    if bv.dtype not in (torch.float64, torch.complex128) or (bv.stride(0) != 1 and bv.stride(1) != 1):
        work = bv.to(torch.complex128 if bv.is_complex() else torch.float64).t().contiguous().t()
    if work.is_complex() and not data.is_complex():
        data = data.to(torch.complex128)  # real factor, complex RHS (rfp.py:101 allows it)
    info = _info(work.device)
    _run(f"rfpk_{_prefix(data.dtype)}pftrs_ex", _capi.flag(desc.transr), _capi.flag(desc.uplo),
         desc.n, work.shape[1], data.data_ptr(), work.data_ptr(), work.stride(0), work.stride(1),
         info.data_ptr(), _capi.stream_handle(work.device))
    if work is not bv:
        bv.copy_(work)
    if foreign is not None:
        host = bv.reshape(tuple(foreign.shape)).cpu()
        if isinstance(foreign, torch.Tensor):
            foreign.copy_(host)
        else:
            foreign[...] = host.numpy()


def tftri(r: RfpTriangle, diag: str = "N") -> int:
    """Invert the RFP-stored triangular factor in place (rfp.py:286-325).
    Returns 0 or the 1-based global index of a zero diagonal entry."""
    diag = normalize_flag(diag, "NU", "diag")
    desc = r.desc
    if desc.n == 0:
        return 0
    info = _info(r.data.device)
    _run(f"rfpk_{_prefix(r.dtype)}tftri", _capi.flag(desc.transr), _capi.flag(desc.uplo),
         _capi.flag(diag), desc.n, r.data.data_ptr(), info.data_ptr(),
         _capi.stream_handle(r.data.device))
    v = int(info.item())
    if v == 0 and r.state is FactorState.CHOLESKY:
        r.state = FactorState.TRIANGULAR_INVERSE
    return v


def pftri(r: RfpTriangle) -> int:
    """Inverse of the SPD/HPD matrix from its Cholesky factor, in place
    (rfp.py:328-360): tftri then the lauum/syrk/trmm stage."""
    if r.state is not FactorState.CHOLESKY:
        raise ValueError(f"pftri needs a Cholesky factor, state is {r.state.value}")
    desc = r.desc
    if desc.n == 0:
        r.state = FactorState.FULL_INVERSE
        return 0
    info = _info(r.data.device)
    _run(f"rfpk_{_prefix(r.dtype)}pftri", _capi.flag(desc.transr), _capi.flag(desc.uplo), desc.n,
         r.data.data_ptr(), info.data_ptr(), _capi.stream_handle(r.data.device))
    v = int(info.item())
    if v == 0:
        r.state = FactorState.FULL_INVERSE
    return v


# ---------------------------------------------------------------- SURVEY 8(f) rows


def _flag(value, allowed, what):
    f = str(value).upper()[:1]
    if f not in allowed:
        raise ValueError(f"{what} must be one of {tuple(allowed)}, got {value!r}")
    return f


def _canon_transr(t):
    return "T" if t == "C" else t


def _check_desc(desc, n, uplo, transr):
    if (desc.n, desc.uplo, desc.transr) != (int(n), uplo, _canon_transr(transr)):
        raise ValueError(
            f"descriptor (n={desc.n}, uplo={desc.uplo}, transr={desc.transr}) "
            f"does not match (n={n}, uplo={uplo}, transr={transr})")


def _device_inplace(b):
    """(working CUDA tensor with a unit stride, foreign original or None)."""
    foreign = None
    if not isinstance(b, torch.Tensor) or not b.is_cuda:
        foreign = b
        bt = as_device(b)
    else:
        bt = b
    work = bt
    if bt.dtype not in (torch.float64, torch.complex128) or (bt.dim() == 2 and bt.stride(0) != 1
                                                            and bt.stride(1) != 1):
        work = bt.to(torch.complex128 if bt.is_complex() else torch.float64).t().contiguous().t()
    return bt, work, foreign


def _writeback(bt, work, foreign):
    if work is not bt:
        bt.copy_(work)
    if foreign is not None:
        host = bt.cpu()
        if isinstance(foreign, torch.Tensor):
            foreign.copy_(host)
        else:
            foreign[...] = host.numpy()


def tfsm(transr: str, side: str, uplo: str, trans: str, diag: str, m: int, n: int, alpha,
         a: RfpTriangle, b) -> None:
    """Triangular solve with an RFP-stored triangle (rfp.py:181-224):
    ``op(A) X = alpha B`` (side 'L') or ``X op(A) = alpha B`` (side 'R'),
    in place on the ``m x n`` array ``b``.  A zero diagonal (diag 'N') raises
    ``kernels.SingularMatrixError`` with the 1-based global index."""
    from .kernels import SingularMatrixError
    transr = _flag(transr, "NTC", "transr")
    side = _flag(side, "LR", "side")
    uplo = _flag(uplo, "LU", "uplo")
    trans = _flag(trans, "NTC", "trans")
    diag = _flag(diag, "NU", "diag")
    order = m if side == "L" else n
    _check_desc(a.desc, order, uplo, transr)
    bt, work, foreign = _device_inplace(b)
    if tuple(bt.shape) != (m, n):
        raise ValueError(f"b must be {(m, n)}, got {tuple(bt.shape)}")
    if m == 0 or n == 0:
        return
    data = a.data
    if work.is_complex() and not data.is_complex():
        data = data.to(torch.complex128)
    if data.is_complex() and not work.is_complex():
        raise ValueError("complex triangle needs a complex right-hand side")
    info = _info(work.device)
    st = _capi.stream_handle(work.device)
    flags = [_capi.flag(x) for x in (a.desc.transr, side, uplo, trans, diag)]
    if data.is_complex():
        al = complex(alpha)
        _run("rfpk_ztfsm", *flags, m, n, al.real, al.imag, data.data_ptr(), work.data_ptr(),
             work.stride(0), work.stride(1), info.data_ptr(), st)
    else:
        _run("rfpk_dtfsm", *flags, m, n, float(alpha), data.data_ptr(), work.data_ptr(),
             work.stride(0), work.stride(1), info.data_ptr(), st)
    v = int(info.item())
    if v:
        raise SingularMatrixError(v)
    _writeback(bt, work, foreign)


def sfrk_hfrk(transr: str, uplo: str, trans: str, n: int, k: int, alpha: float, a, beta: float,
              c: RfpTriangle, hermitian=None) -> None:
    """RFP rank-k update ``C <- alpha G G^(T|H) + beta C`` (rfp.py:227-283),
    G = A (n x k) for trans 'N', A^(T|H) (A k x n) otherwise; real alpha, beta."""
    transr = _flag(transr, "NTC", "transr")
    uplo = _flag(uplo, "LU", "uplo")
    trans = _flag(trans, "NTC", "trans")
    _check_desc(c.desc, n, uplo, transr)
    alpha, beta = float(alpha), float(beta)
    herm = c.data.is_complex() if hermitian is None else bool(hermitian)
    if c.data.is_complex() and not herm:
        raise ValueError("complex symmetric (non-conjugated) updates are not supported")
    if n == 0:
        return
    st = _capi.stream_handle(c.data.device)
    flags = [_capi.flag(x) for x in (c.desc.transr, uplo, trans)]
    if alpha == 0 or k == 0:
        if c.data.is_complex():
            _run("rfpk_zhfrk", *flags, n, 0, 0.0, 0, 1, 1, beta, c.data.data_ptr(), 1, st)
        else:
            _run("rfpk_dsfrk", *flags, n, 0, 0.0, 0, 1, 1, beta, c.data.data_ptr(), st)
        return
    at = as_device(a)
    want = (n, k) if trans == "N" else (k, n)
    if tuple(at.shape) != want:
        raise ValueError(f"a must be {want} for trans={trans!r}, got {tuple(at.shape)}")
    if at.stride(0) != 1 and at.stride(1) != 1:
        at = at.t().contiguous().t()
    if c.data.is_complex():
        at = at.to(torch.complex128)
        _run("rfpk_zhfrk", *flags, n, k, alpha, at.data_ptr(), at.stride(0), at.stride(1), beta,
             c.data.data_ptr(), 1, st)
    else:
        if at.is_complex():
            raise ValueError("real triangle needs a real update matrix")
        _run("rfpk_dsfrk", *flags, n, k, alpha, at.data_ptr(), at.stride(0), at.stride(1), beta,
             c.data.data_ptr(), st)


def lansf(norm: str, r: RfpTriangle, hermitian: bool = True) -> float:
    """Norm of the full symmetric/Hermitian matrix implied by an RFP triangle
    (rfp.py:363-417): 'M' max |a|, '1'/'O' and 'I' (equal for symmetric),
    'F'/'E' Frobenius.  One device pass over the RFP buffer."""
    nm = str(norm).upper()[:1]
    if nm not in ("M", "1", "O", "I", "F", "E"):
        raise ValueError(f"unknown norm selector {nm!r}")
    d = r.desc
    if d.n == 0:
        return 0.0
    out = torch.zeros(1, dtype=torch.float64, device=r.data.device)
    fn = "rfpk_zlansf" if r.data.is_complex() else "rfpk_dlansf"
    _run(fn, _capi.flag(nm), _capi.flag(d.transr), _capi.flag(d.uplo), d.n, r.data.data_ptr(),
         out.data_ptr(), _capi.stream_handle(r.data.device))
    return float(out.item())


# ---------------------------------------------------------------- batched


def _batched_args(arf, n, uplo, transr):
    desc = make_descriptor(n, uplo, transr)
    if not isinstance(arf, torch.Tensor) or not arf.is_cuda or arf.dtype != torch.float64:
        raise ValueError("arf must be a float64 CUDA tensor of shape (batch, nt)")
    if arf.dim() != 2 or arf.shape[1] != desc.nt or arf.stride(1) != 1:
        raise ValueError(f"arf must be (batch, {desc.nt}) with unit inner stride")
    return desc


def _batched_rhs(b, desc, batch):
    if not isinstance(b, torch.Tensor) or not b.is_cuda or b.dtype != torch.float64:
        raise ValueError("b must be a float64 CUDA tensor")
    bv = b.unsqueeze(-1) if b.dim() == 2 else b
    if bv.dim() != 3 or bv.shape[0] != batch or bv.shape[1] != desc.n:
        raise ValueError(f"b must be (batch, {desc.n}[, nrhs]), got {tuple(b.shape)}")
    work = bv if bv.stride(1) == 1 else bv.transpose(1, 2).contiguous().transpose(1, 2)
    ldb = work.stride(2) if work.shape[2] > 1 else max(desc.n, 1)
    return bv, work, ldb


def pftrf_batched(arf: torch.Tensor, transr: str, uplo: str, n: int) -> torch.Tensor:
    """pftrf on ``batch`` independent RFP buffers (rows of ``arf``), in place,
    LAPACK argument order (``pftrf_batched(arf[batch, nt],
    transr, uplo, n) -> info[batch]``).  Returns the per-matrix info as an
    int32 CUDA tensor (no host sync)."""
    desc = _batched_args(arf, n, uplo, transr)
    batch = arf.shape[0]
    info = torch.empty(batch, dtype=torch.int32, device=arf.device)
    _run("rfpk_dpftrf_batched", _capi.flag(desc.transr), _capi.flag(desc.uplo), n,
         arf.data_ptr(), arf.stride(0), batch, info.data_ptr(), _capi.stream_handle(arf.device))
    return info


def pftrs_batched(arf: torch.Tensor, transr: str, uplo: str, n: int, b: torch.Tensor) -> None:
    """pftrs for each factor ``arf[k]`` against ``b[k]`` ((batch, n) or
    (batch, n, nrhs)), in place on ``b``."""
    desc = _batched_args(arf, n, uplo, transr)
    batch = arf.shape[0]
    bv, work, ldb = _batched_rhs(b, desc, batch)
    info = torch.empty(batch, dtype=torch.int32, device=arf.device)
    _run("rfpk_dpftrs_batched", _capi.flag(desc.transr), _capi.flag(desc.uplo), n, work.shape[2],
         arf.data_ptr(), arf.stride(0), work.data_ptr(), ldb, work.stride(0), batch,
         info.data_ptr(), _capi.stream_handle(arf.device))
    if work is not bv:
        bv.copy_(work)


def pftrf_pftrs_batched(arf: torch.Tensor, transr: str, uplo: str, n: int,
                        b: torch.Tensor) -> torch.Tensor:
    """Fused pftrf + pftrs over a batch (one HBM pass per matrix)."""
    desc = _batched_args(arf, n, uplo, transr)
    batch = arf.shape[0]
    bv, work, ldb = _batched_rhs(b, desc, batch)
    info = torch.empty(batch, dtype=torch.int32, device=arf.device)
    _run("rfpk_dpftrf_pftrs_batched", _capi.flag(desc.transr), _capi.flag(desc.uplo), n,
         work.shape[2], arf.data_ptr(), arf.stride(0), work.data_ptr(), ldb, work.stride(0),
         batch, info.data_ptr(), _capi.stream_handle(arf.device))
    if work is not bv:
        bv.copy_(work)
    return info


def pftrf_pftrs_batched_from_host(host_arf: torch.Tensor, transr: str, uplo: str, n: int,
                                  host_b: torch.Tensor, out=None, chunk: int = 4096):
    """:func:`pftrf_pftrs_batched` for a batch that sits in (pinned) host
    memory, pipelined in chunks of ``chunk`` matrices over three streams: the
    host->device copy of chunk k+1 and the device->host copy of chunk k-1's
    solutions overlap the fused kernel on chunk k (PCIe is full duplex), so
    the call approaches the pure transfer time.  ``host_arf``: (batch, nt)
    float64; ``host_b``: (batch, n) or (batch, n, nrhs) float64 with unit
    stride along n.  Solutions go to ``out`` (default ``host_b``).  Returns
    ``(arf on the device holding the factors, info)``; info is an int32 CUDA
    tensor, valid once the current stream reaches it (no host sync here)."""
    desc = make_descriptor(n, uplo, transr)
    if not isinstance(host_arf, torch.Tensor) or host_arf.is_cuda or host_arf.dtype != torch.float64:
        raise ValueError("host_arf must be a float64 CPU tensor of shape (batch, nt)")
    if host_arf.dim() != 2 or host_arf.shape[1] != desc.nt or host_arf.stride(1) != 1:
        raise ValueError(f"host_arf must be (batch, {desc.nt}) with unit inner stride")
    batch = host_arf.shape[0]
    if not isinstance(host_b, torch.Tensor) or host_b.is_cuda or host_b.dtype != torch.float64:
        raise ValueError("host_b must be a float64 CPU tensor")
    hb = host_b.unsqueeze(-1) if host_b.dim() == 2 else host_b
    if hb.dim() != 3 or hb.shape[0] != batch or hb.shape[1] != n or (n > 1 and hb.stride(1) != 1):
        raise ValueError(f"host_b must be (batch, {n}[, nrhs]) with unit stride along n")
    ho = hb if out is None else (out.unsqueeze(-1) if out.dim() == 2 else out)
    if ho.shape != hb.shape or ho.stride() != hb.stride():
        raise ValueError("out must match host_b's shape and strides")
    if chunk < 1:
        raise ValueError("chunk must be positive")
    dev = torch.device("cuda", torch.cuda.current_device())
    main = torch.cuda.current_stream(dev)
    s_in, s_out = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    d_arf = torch.empty((batch, desc.nt), dtype=torch.float64, device=dev)
    d_b = torch.empty_strided(hb.shape, hb.stride(), dtype=torch.float64, device=dev)
    infos = []
    s_in.wait_stream(main)
    s_out.wait_stream(main)
    for k0 in range(0, batch, chunk):
        k1 = min(batch, k0 + chunk)
        with torch.cuda.stream(s_in):
            d_arf[k0:k1].copy_(host_arf[k0:k1], non_blocking=True)
            d_b[k0:k1].copy_(hb[k0:k1], non_blocking=True)
        main.wait_stream(s_in)
        with torch.cuda.stream(main):
            infos.append(pftrf_pftrs_batched(d_arf[k0:k1], transr, uplo, n, d_b[k0:k1]))
        s_out.wait_stream(main)
        with torch.cuda.stream(s_out):
            ho[k0:k1].copy_(d_b[k0:k1], non_blocking=True)
    main.wait_stream(s_out)
    for t in (d_arf, d_b):
        t.record_stream(s_in)
        t.record_stream(s_out)
    info = torch.cat(infos) if infos else torch.empty(0, dtype=torch.int32, device=dev)
    return d_arf, info
