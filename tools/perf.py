"""Developer perf sweep (run under gpurun): times each BASELINE config's
operations and the core kernels with CUDA events.  Not the bench contract
(that is bench.py); prints one JSON object per line."""

import argparse
import ctypes
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_0901_1696_b200 import _capi  # noqa: E402

lib = _capi.lib()
dev = torch.device("cuda:0")
PEAK = 37.2e12  # nominal FP64 (148 SM x 128 flop/clk x 1.965 GHz)


def ev_time(fn, reps=5, setup=None):
    ts = []
    for i in range(reps + 1):
        if setup:
            setup()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        if i:
            ts.append(s.elapsed_time(e))
    return float(np.median(ts))


def st():
    return _capi.stream_handle(dev)


def spd_gpu(n, cplx=False, seed=0, scale="1/n"):
    g = torch.Generator(device=dev).manual_seed(seed)
    if cplx:
        b = torch.randn(n, n, dtype=torch.complex128, device=dev, generator=g)
    else:
        b = torch.randn(n, n, dtype=torch.float64, device=dev, generator=g)
    a = b @ b.mH
    if scale == "1/n":
        a /= n
        a.diagonal().add_(1.0)
    else:
        a.diagonal().add_(float(n))
    return a  # symmetric => also column-major-valid


def out(**kw):
    print(json.dumps(kw), flush=True)


def gemm_bench():
    for (m, n, k) in [(8192, 8192, 8192), (4096, 4096, 4096), (8192, 1024, 8192), (2000, 64, 2000)]:
        for ta, tb in [("N", "N"), ("T", "N"), ("N", "T")]:
            a = torch.randn(k, m, dtype=torch.float64, device=dev).t() if ta == "N" else torch.randn(m, k, dtype=torch.float64, device=dev).t()
            b = torch.randn(n, k, dtype=torch.float64, device=dev).t() if tb == "N" else torch.randn(k, n, dtype=torch.float64, device=dev).t()
            c = torch.randn(n, m, dtype=torch.float64, device=dev).t()
            def run():
                lib.rfpk_dgemm(ta.encode(), tb.encode(), -1.0, a.data_ptr(), a.shape[0], a.shape[1], a.stride(0), a.stride(1),
                               b.data_ptr(), b.shape[0], b.shape[1], b.stride(0), b.stride(1), 1.0,
                               c.data_ptr(), m, n, c.stride(0), c.stride(1), st())
            ms = ev_time(run, 5)
            out(kind="dgemm", m=m, n=n, k=k, ta=ta, tb=tb, ms=ms, tflops=2 * m * n * k / ms / 1e9)
    # odd leading dimension (real TRANSR='N' RFP blocks)
    n = 8192
    base = torch.randn(n + 1, 3 * n, dtype=torch.float64, device=dev)
    A = base.t()[: n, :n]  # not our layout; build col-major with ld n+1
    buf = torch.randn((n + 1) * n * 3, dtype=torch.float64, device=dev)
    a = buf[: (n + 1) * n].view(n, n + 1).t()[:n]
    b = buf[(n + 1) * n: 2 * (n + 1) * n].view(n, n + 1).t()[:n]
    c = buf[2 * (n + 1) * n:].view(n, n + 1).t()[:n]
    def run():
        lib.rfpk_dgemm(b"N", b"T", -1.0, a.data_ptr(), n, n, a.stride(0), a.stride(1),
                       b.data_ptr(), n, n, b.stride(0), b.stride(1), 1.0, c.data_ptr(), n, n, c.stride(0), c.stride(1), st())
    ms = ev_time(run, 5)
    out(kind="dgemm_oddld", n=n, ms=ms, tflops=2 * n ** 3 / ms / 1e9)
    for cn in (4096,):
        a = torch.randn(cn, cn, dtype=torch.complex128, device=dev)
        b = torch.randn(cn, cn, dtype=torch.complex128, device=dev)
        c = torch.randn(cn, cn, dtype=torch.complex128, device=dev)
        def runz():
            lib.rfpk_zgemm(b"N", b"N", -1.0, 0.0, a.data_ptr(), cn, cn, 1, cn, b.data_ptr(), cn, cn, 1, cn, 1.0, 0.0,
                           c.data_ptr(), cn, cn, 1, cn, st())
        ms = ev_time(runz, 3)
        out(kind="zgemm", n=cn, ms=ms, tflops=8 * cn ** 3 / ms / 1e9)


def rfp_bench(n, uplo, transr, nrhs, do_pftri=False, cplx=False, reps=5):
    from paper_0901_1696_b200 import convert
    a = spd_gpu(n, cplx, seed=n)
    r = convert.trttf(a, uplo, transr)
    del a
    saved = r.data.clone()
    info = torch.zeros(1, dtype=torch.int32, device=dev)
    p = "z" if cplx else "d"
    f_pftrf = getattr(lib, f"rfpk_{p}pftrf")
    def setup():
        r.data.copy_(saved)
    def run():
        f_pftrf(transr.encode(), uplo.encode(), n, r.data.data_ptr(), info.data_ptr(), st())
    ms = ev_time(run, reps, setup)
    mul = 4 if cplx else 1
    res = dict(kind="pftrf", n=n, uplo=uplo, transr=transr, dtype=p, ms=ms,
               tflops=mul * n ** 3 / 3 / ms / 1e9, info=int(info.item()))
    res["frac_nominal"] = res["tflops"] * 1e12 / PEAK
    out(**res)
    if nrhs:
        dt = torch.complex128 if cplx else torch.float64
        b0 = torch.randn(nrhs, n, dtype=dt, device=dev).t()
        b = b0.clone()
        f_pftrs = getattr(lib, f"rfpk_{p}pftrs")
        def setb():
            b.copy_(b0)
        def runs():
            f_pftrs(transr.encode(), uplo.encode(), n, nrhs, r.data.data_ptr(), b.data_ptr(), n, info.data_ptr(), st())
        ms = ev_time(runs, reps, setb)
        out(kind="pftrs", n=n, nrhs=nrhs, uplo=uplo, transr=transr, dtype=p, ms=ms,
            tflops=mul * 2 * n * n * nrhs / ms / 1e9)
    if do_pftri:
        fac = r.data.clone()
        f_pftri = getattr(lib, f"rfpk_{p}pftri")
        def setf():
            r.data.copy_(fac)
        def runi():
            f_pftri(transr.encode(), uplo.encode(), n, r.data.data_ptr(), info.data_ptr(), st())
        ms = ev_time(runi, reps, setf)
        out(kind="pftri", n=n, uplo=uplo, transr=transr, dtype=p, ms=ms,
            tflops=mul * 2 * n ** 3 / 3 / ms / 1e9, info=int(info.item()))


def conv_bench(n, uplos="L", cplx=False, reps=5):
    """Conversions at order n: bytes = every element read once + written once
    (tfttr also writes the zeroed other triangle of the n x n output)."""
    nt = n * (n + 1) // 2
    dt = torch.complex128 if cplx else torch.float64
    es = 16 if cplx else 8
    p = "z" if cplx else "d"
    a = torch.randn(n, n, dtype=dt, device=dev)
    arf = torch.empty(nt, dtype=dt, device=dev)
    pk = torch.empty(nt, dtype=dt, device=dev)
    full = torch.empty(n, n, dtype=dt, device=dev)
    f = lambda name: getattr(lib, f"rfpk_{p}{name}")
    for u in uplos:
        for tr in "NT":
            ms = ev_time(lambda: f("trttf")(tr.encode(), u.encode(), n, a.data_ptr(), n, arf.data_ptr(), st()), reps)
            out(kind="trttf", n=n, uplo=u, transr=tr, dtype=p, ms=ms, gbs=2 * nt * es / ms / 1e6)
            ms = ev_time(lambda: f("tfttr")(tr.encode(), u.encode(), n, arf.data_ptr(), full.data_ptr(), n, st()), reps)
            out(kind="tfttr", n=n, uplo=u, transr=tr, dtype=p, ms=ms, gbs=(nt + n * n) * es / ms / 1e6)
            ms = ev_time(lambda: f("tfttp")(tr.encode(), u.encode(), n, arf.data_ptr(), pk.data_ptr(), st()), reps)
            out(kind="tfttp", n=n, uplo=u, transr=tr, dtype=p, ms=ms, gbs=2 * nt * es / ms / 1e6)
            ms = ev_time(lambda: f("tpttf")(tr.encode(), u.encode(), n, pk.data_ptr(), arf.data_ptr(), st()), reps)
            out(kind="tpttf", n=n, uplo=u, transr=tr, dtype=p, ms=ms, gbs=2 * nt * es / ms / 1e6)


def frows_bench(n=16384, k=8192, nrhs=1024):
    """SURVEY 8(f) rows at config-3 size: lansf (HBM: nt*8 bytes read),
    sfrk (n^2 k flops), tfsm (n^2 nrhs flops)."""
    nt = n * (n + 1) // 2
    arf = torch.randn(nt, dtype=torch.float64, device=dev)
    res = torch.zeros(1, dtype=torch.float64, device=dev)
    for norm in "M1IF":
        ms = ev_time(lambda: lib.rfpk_dlansf(norm.encode(), b"N", b"L", n, arf.data_ptr(), res.data_ptr(), st()), 5)
        out(kind="lansf", norm=norm, n=n, ms=ms, gbs=nt * 8 / ms / 1e6)
    a = torch.randn(k, n, dtype=torch.float64, device=dev).t()  # n x k column-major
    ms = ev_time(lambda: lib.rfpk_dsfrk(b"N", b"L", b"N", n, k, -1.0, a.data_ptr(), 1, n, 1.0, arf.data_ptr(), st()), 3)
    out(kind="sfrk", n=n, k=k, ms=ms, tflops=n * n * k / ms / 1e9)
    g = torch.randn(n, n, dtype=torch.float64, device=dev); s = g @ g.t() / n; s.diagonal().add_(1.0)
    from paper_0901_1696_b200 import convert
    r = convert.trttf(s, "L", "N"); del g, s
    info = torch.zeros(1, dtype=torch.int32, device=dev)
    lib.rfpk_dpftrf(b"N", b"L", n, r.data.data_ptr(), info.data_ptr(), st())
    b0 = torch.randn(nrhs, n, dtype=torch.float64, device=dev).t(); b = b0.clone()
    ms = ev_time(lambda: lib.rfpk_dtfsm(b"N", b"L", b"L", b"N", b"N", n, nrhs, 1.0, r.data.data_ptr(),
                                        b.data_ptr(), 1, n, info.data_ptr(), st()), 3, lambda: b.copy_(b0))
    out(kind="tfsm", n=n, nrhs=nrhs, ms=ms, tflops=n * n * nrhs / ms / 1e9)


def batched_bench(batch=65536, n=64, nrhs=8):
    nt = n * (n + 1) // 2
    from paper_0901_1696_b200 import convert
    a = spd_gpu(n, scale="n")
    one = convert.trttf(a, "U", "N").data
    arf0 = one.unsqueeze(0).repeat(batch, 1).contiguous()
    arf = arf0.clone()
    b0 = torch.randn(batch, nrhs, n, dtype=torch.float64, device=dev)
    b = b0.clone()
    info = torch.zeros(batch, dtype=torch.int32, device=dev)
    def setup():
        arf.copy_(arf0)
        b.copy_(b0)
    def run():
        lib.rfpk_dpftrf_pftrs_batched(b"N", b"U", n, nrhs, arf.data_ptr(), nt, b.data_ptr(), n, n * nrhs, batch,
                                      info.data_ptr(), st())
    ms = ev_time(run, 5, setup)
    byts = batch * (2 * nt * 8 + 2 * n * nrhs * 8)
    out(kind="batched_fused", batch=batch, n=n, nrhs=nrhs, ms=ms, mats_per_s=batch / ms * 1e3,
        gbs=byts / ms / 1e6, info=int(info.abs().sum()))


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--what", default="all")
    args = ap.parse_args()
    w = args.what
    if w in ("all", "gemm"):
        gemm_bench()
    if w == "small":
        rfp_bench(1000, "L", "N", 100, do_pftri=True)
        rfp_bench(300, "L", "N", 100, do_pftri=True)
        rfp_bench(2000, "U", "N", 64, do_pftri=True)
        rfp_bench(4000, "L", "N", 64)
    if w in ("all", "rfp"):
        rfp_bench(1000, "L", "N", 100, do_pftri=True)
        for n in (4000, 4001):
            for u in "LU":
                for t in "NT":
                    rfp_bench(n, u, t, 64)
        rfp_bench(16384, "L", "N", 1024, reps=3)
    if w == "mid":
        for n in (1000, 2000, 3000, 4000, 4001, 6000, 8000, 8193):
            for u in "LU":
                for t in "NT":
                    rfp_bench(n, u, t, 64, reps=5)
    if w == "big":
        rfp_bench(16384, "L", "N", 1024, reps=3)
        rfp_bench(4000, "L", "N", 64)
    if w in ("all", "cplx"):
        rfp_bench(6000, "L", "T", 0, do_pftri=True, cplx=True, reps=2)
    if w in ("all", "conv"):
        conv_bench(16384)
    if w in ("all", "frows"):
        frows_bench()
    if w == "convall":
        conv_bench(16384, "LU")
        conv_bench(16383, "LU")
        conv_bench(11584, "L", cplx=True)
    if w in ("all", "batched"):
        batched_bench()
