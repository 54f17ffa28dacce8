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

import torch

from . import _capi
from .convert import FactorState, RfpTriangle, _prefix, as_device
from .layout import make_descriptor, normalize_flag

__all__ = [
    "pftrf",
    "pftrs",
    "tftri",
    "pftri",
    "pftrf_batched",
    "pftrs_batched",
    "pftrf_pftrs_batched",
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


def pftrf_batched(arf: torch.Tensor, n: int, uplo: str = "U", transr: str = "N") -> torch.Tensor:
    """pftrf on ``batch`` independent RFP buffers (rows of ``arf``), in place.
    Returns the per-matrix info as an int32 CUDA tensor (no host sync)."""
    desc = _batched_args(arf, n, uplo, transr)
    batch = arf.shape[0]
    info = torch.empty(batch, dtype=torch.int32, device=arf.device)
    _run("rfpk_dpftrf_batched", _capi.flag(desc.transr), _capi.flag(desc.uplo), n,
         arf.data_ptr(), arf.stride(0), batch, info.data_ptr(), _capi.stream_handle(arf.device))
    return info


def pftrs_batched(arf: torch.Tensor, b: torch.Tensor, n: int, uplo: str = "U",
                  transr: str = "N") -> None:
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


def pftrf_pftrs_batched(arf: torch.Tensor, b: torch.Tensor, n: int, uplo: str = "U",
                        transr: str = "N") -> torch.Tensor:
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
