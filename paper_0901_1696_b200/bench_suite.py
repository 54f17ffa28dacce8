"""The SPEC bench record: factor /
solve / invert timed in full, packed and RFP storage on the GPU through this
package's public calls, one ``BenchRecord`` per (routine, format, n, uplo,
transr), written as CSV with the exact header

    routine,format,n,nrhs,uplo,transr,reps,median_seconds,mflops,residual,seed

Methodology: the SPD input is built
once on the host from the seed (A = B B^T + n I, B ~ N(0,1),
``numpy.random.default_rng(seed)`` as the reference's generator convention);
every rep restores the input (untimed) and times ONLY the routine call with
CUDA events; ``median_seconds`` is the median over ``reps``; ``mflops`` =
flop model / median / 1e6 with n^3/3 (factor), 2 n^2 nrhs (solve), 2 n^3/3
(invert); ``residual`` is the inline check, scaled by n * eps:
factor ||A - L L^T||_F / (n eps ||A||_F), solve ||A X - B||_F / (n eps ||A||_F
||X||_F), invert ||A A^-1 - I||_F / (n eps ||A||_F ||A^-1||_F).  A record
whose residual exceeds ``tol`` fails the run (exit status 1) unless
``keep_going``.

Formats: ``rfp`` = pftrf / pftrs / pftri (every TRANSR), ``packed`` =
pptrf_ref / pptrs_ref (the reference has no packed inverse: no invert
record), ``full`` = the library's full-storage potrf, the potrs pair of
triangular solves and potri = trtri + lauum (kernels.py).

    python -m paper_0901_1696_b200.bench_suite --sizes 500,1000 --out bench.csv
"""

from __future__ import annotations

import argparse
import csv
import math
import sys
from dataclasses import dataclass

import numpy as np

HEADER = ["routine", "format", "n", "nrhs", "uplo", "transr", "reps", "median_seconds", "mflops",
          "residual", "seed"]
ROUTINES = ("factor", "solve", "invert")
FORMATS = ("full", "packed", "rfp")
EPS = 2.0 ** -53


@dataclass
class BenchRecord:
    routine: str
    format: str
    n: int
    nrhs: int
    uplo: str
    transr: str  # "" for full / packed
    reps: int
    median_seconds: float
    mflops: float
    residual: float
    seed: int
    failed: bool = False


def flop_model(routine: str, n: int, nrhs: int) -> float:
    """LAPACK-conventional leading terms."""
    if routine == "factor":
        return n ** 3 / 3.0
    if routine == "solve":
        return 2.0 * n * n * nrhs
    return 2.0 * n ** 3 / 3.0


def nrhs_for(n: int, rule: str, fixed: int) -> int:
    """``fixed`` (the Tigerton captions: 100) or ``max(100, n/10)`` (PAPER.md
    figure captions)."""
    return max(100, n // 10) if rule == "max" else fixed


def spd(n: int, seed: int) -> np.ndarray:
    rng = np.random.default_rng(seed)
    b = rng.standard_normal((n, n))
    a = b @ b.T
    a[np.diag_indices(n)] += n
    return np.asfortranarray(a)


def _timed(torch, setup, call, reps):
    """median seconds of ``call`` over ``reps`` runs, each after ``setup``
    (outside the CUDA-event bracket)."""
    ts = []
    for _ in range(reps):
        state = setup()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        out = call(state)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / 1e3)
    return float(np.median(ts)), state, out


def _fro(t):
    return float(t.norm())


def run_case(routine, fmt, n, nrhs, uplo, transr, reps, seed, a_host=None):
    """One BenchRecord (or None when the format has no such routine)."""
    import torch

    from . import convert, kernels, packed, rfp

    if fmt == "packed" and routine == "invert":
        return None
    a_host = spd(n, seed) if a_host is None else a_host
    dev = torch.device("cuda")
    a = torch.from_numpy(a_host).to(dev)
    anorm = _fro(a)
    rng = np.random.default_rng(seed + 1)
    b_host = np.asfortranarray(rng.standard_normal((n, nrhs)))
    lower = uplo == "L"

    # the factored input for solve / invert (untimed)
    def factored():
        if fmt == "rfp":
            r = convert.trttf(a, uplo, transr)
            assert rfp.pftrf(r) == 0
            return r
        if fmt == "packed":
            p = packed.pack(a, uplo)
            assert packed.pptrf_ref(p) == 0
            return p
        f = a.t().contiguous().t().clone()  # column-major copy
        assert kernels.potrf_ref(uplo, f) == 0
        return f

    def full_factor(obj):
        """the triangular factor as a full tensor (zeros elsewhere)"""
        if fmt == "rfp":
            t = convert.tfttr(obj)
        elif fmt == "packed":
            t = packed.unpack(obj)
        else:
            t = obj
        return torch.tril(t) if lower else torch.triu(t)

    if routine == "factor":
        if fmt == "rfp":
            base = convert.trttf(a, uplo, transr)
            sec, obj, info = _timed(torch, lambda: base.copy(), rfp.pftrf, reps)
        elif fmt == "packed":
            base = packed.pack(a, uplo)
            sec, obj, info = _timed(
                torch, lambda: convert.PackedTriangle(base.data.clone(), n, uplo),
                packed.pptrf_ref, reps)
        else:
            base = a.t().contiguous().t()
            sec, obj, info = _timed(torch, lambda: base.clone(),
                                    lambda f: kernels.potrf_ref(uplo, f), reps)
        f = full_factor(obj)
        rec = f @ f.t() if lower else f.t() @ f
        res = _fro(rec - a) / (n * EPS * anorm) if info == 0 else math.inf
    elif routine == "solve":
        obj = factored()
        bt = torch.from_numpy(b_host).to(dev)

        def setup():
            return bt.t().contiguous().t().clone()

        if fmt == "rfp":
            sec, x, _ = _timed(torch, setup, lambda x: rfp.pftrs(obj, x), reps)
        elif fmt == "packed":
            sec, x, _ = _timed(torch, setup, lambda x: packed.pptrs_ref(obj, x), reps)
        else:
            def potrs(x):
                if lower:
                    kernels.trsm("L", "L", "N", "N", 1.0, obj, x)
                    kernels.trsm("L", "L", "C", "N", 1.0, obj, x)
                else:
                    kernels.trsm("L", "U", "C", "N", 1.0, obj, x)
                    kernels.trsm("L", "U", "N", "N", 1.0, obj, x)
            sec, x, _ = _timed(torch, setup, potrs, reps)
        res = _fro(a @ x - bt) / (n * EPS * anorm * _fro(x))
    else:  # invert
        if fmt == "rfp":
            base = factored()
            sec, obj, info = _timed(torch, lambda: base.copy(), rfp.pftri, reps)
            inv = convert.tfttr(obj)
        else:
            base = factored()

            def potri(f):
                kernels.trtri_ref(uplo, "N", f)
                kernels.lauum_ref(uplo, f)
                return 0
            sec, obj, info = _timed(torch, lambda: base.clone(), potri, reps)
            inv = obj
        tri = torch.tril(inv) if lower else torch.triu(inv)
        inv = tri + tri.t() - torch.diag(torch.diagonal(tri))
        res = (_fro(a @ inv - torch.eye(n, dtype=a.dtype, device=dev))
               / (n * EPS * anorm * _fro(inv))) if info == 0 else math.inf
    fl = flop_model(routine, n, nrhs)
    return BenchRecord(routine, fmt, n, nrhs if routine == "solve" else 0, uplo,
                       transr if fmt == "rfp" else "", reps, sec, fl / sec / 1e6, res, seed)


def run_suite(sizes, routines=ROUTINES, formats=FORMATS, uplos="LU", transrs="NT",
              nrhs_rule="fixed", nrhs=100, reps=5, seed=0, tol=10.0, keep_going=False):
    """Every (size, format, routine, uplo[, transr]) combination; returns the
    records.  Raises RuntimeError on the first failed
    residual unless ``keep_going`` (failed records are then marked)."""
    if not sizes:
        raise ValueError("sizes must be nonempty")
    if reps < 3:
        raise ValueError("reps must be >= 3")
    out = []
    for n in sizes:
        a_host = spd(n, seed)
        k = nrhs_for(n, nrhs_rule, nrhs)
        for fmt in formats:
            for routine in routines:
                for uplo in uplos:
                    for transr in (transrs if fmt == "rfp" else ("",)):
                        r = run_case(routine, fmt, n, k, uplo, transr, reps, seed, a_host)
                        if r is None:
                            continue
                        if not (r.residual <= tol):
                            r.failed = True
                            if not keep_going:
                                raise RuntimeError(f"residual check failed: {r}")
                        out.append(r)
    return out


def _fmt(v):
    return repr(float(v)) if isinstance(v, float) else str(v)


def emit_csv(records, path) -> None:
    """Header row exactly ``HEADER``, one row per record, LF line endings,
    '.' decimals, 17 significant digits (round-trip exact)."""
    with open(path, "w", newline="", encoding="utf-8") as f:
        w = csv.writer(f, lineterminator="\n")
        w.writerow(HEADER)
        for r in records:
            w.writerow([r.routine, r.format, r.n, r.nrhs, r.uplo, r.transr, r.reps,
                        f"{r.median_seconds:.17g}", f"{r.mflops:.17g}", f"{r.residual:.17g}",
                        r.seed])


def read_csv(path):
    """Parse a file written by emit_csv back into BenchRecords."""
    with open(path, newline="", encoding="utf-8") as f:
        rows = list(csv.reader(f))
    if not rows or rows[0] != HEADER:
        raise ValueError("not a bench CSV (header mismatch)")
    return [BenchRecord(r[0], r[1], int(r[2]), int(r[3]), r[4], r[5], int(r[6]), float(r[7]),
                        float(r[8]), float(r[9]), int(r[10])) for r in rows[1:]]


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="python -m paper_0901_1696_b200.bench_suite")
    ap.add_argument("--sizes", default="50,100,200,400,500,800,1000,1600,2000")
    ap.add_argument("--routines", default=",".join(ROUTINES))
    ap.add_argument("--formats", default=",".join(FORMATS))
    ap.add_argument("--uplo", default="LU")
    ap.add_argument("--transr", default="NT")
    ap.add_argument("--nrhs", type=int, default=100)
    ap.add_argument("--nrhs-rule", choices=["fixed", "max"], default="fixed")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--out", default="bench.csv")
    ap.add_argument("--keep-going", action="store_true")
    try:
        args = ap.parse_args(argv)
    except SystemExit as e:
        return 64 if e.code else 0
    sizes = [int(s) for s in args.sizes.split(",") if s]
    for name, vals, allowed in (("routines", args.routines.split(","), ROUTINES),
                                ("formats", args.formats.split(","), FORMATS)):
        bad = [v for v in vals if v not in allowed]
        if bad:
            print(f"unknown {name}: {bad}", file=sys.stderr)
            return 64
    try:
        recs = run_suite(sizes, args.routines.split(","), args.formats.split(","),
                         args.uplo.upper(), args.transr.upper(), args.nrhs_rule, args.nrhs,
                         args.reps, args.seed, keep_going=args.keep_going)
    except RuntimeError as e:
        print(e, file=sys.stderr)
        return 1
    try:
        emit_csv(recs, args.out)
    except OSError as e:
        print(e, file=sys.stderr)
        return 2
    return 1 if any(r.failed for r in recs) else 0


if __name__ == "__main__":
    sys.exit(main())
