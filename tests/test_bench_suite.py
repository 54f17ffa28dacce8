"""The SPEC bench record:
paper_0901_1696_b200.bench_suite.  CPU tests cover the CSV format, the flop
model, the nrhs rule and the CLI's argument errors; the GPU test runs a small
suite over every format and checks the records."""

import math
import os

import pytest

from paper_0901_1696_b200 import bench_suite as B


def _rec(**kw):
    base = dict(routine="factor", format="rfp", n=50, nrhs=0, uplo="L", transr="N", reps=3,
                median_seconds=1.2345678901234567e-4, mflops=337.50000000000006,
                residual=0.12345678901234568, seed=7)
    base.update(kw)
    return B.BenchRecord(**base)


def test_csv_header_and_round_trip(tmp_path):
    """Header row exactly as SPEC.md:399; LF endings; 17 significant digits so
    the parse-back recovers every field bit-exactly; empty -> header only."""
    p = tmp_path / "b.csv"
    B.emit_csv([], p)
    assert p.read_bytes() == (",".join(B.HEADER) + "\n").encode()
    assert p.read_text().strip() == ("routine,format,n,nrhs,uplo,transr,reps,median_seconds,"
                                     "mflops,residual,seed")
    recs = [_rec(), _rec(routine="solve", format="packed", nrhs=100, uplo="U", transr="",
                         median_seconds=3.0e-3, mflops=1.0 / 3.0, residual=math.pi, seed=2**63 - 1)]
    B.emit_csv(recs, p)
    raw = p.read_bytes()
    assert b"\r" not in raw and raw.count(b"\n") == 3
    back = B.read_csv(p)
    for a, b in zip(recs, back):
        for f in ("routine", "format", "n", "nrhs", "uplo", "transr", "reps", "seed"):
            assert getattr(a, f) == getattr(b, f)
        for f in ("median_seconds", "mflops", "residual"):
            assert getattr(a, f) == getattr(b, f)  # bit-exact through 17 digits


def test_flop_model_and_nrhs_rule():
    assert B.flop_model("factor", 30, 0) == 30 ** 3 / 3
    assert B.flop_model("solve", 30, 7) == 2 * 30 * 30 * 7
    assert B.flop_model("invert", 30, 0) == 2 * 30 ** 3 / 3
    assert B.nrhs_for(2000, "max", 100) == 200   # SPEC.md:396 example
    assert B.nrhs_for(500, "max", 100) == 100
    assert B.nrhs_for(2000, "fixed", 100) == 100


def test_cli_argument_errors():
    assert B.main(["--bogus-flag"]) == 64
    assert B.main(["--routines", "factor,dance"]) == 64
    assert B.main(["--formats", "banded"]) == 64
    with pytest.raises(ValueError):
        B.run_suite([], reps=3)
    with pytest.raises(ValueError):
        B.run_suite([50], reps=2)


@pytest.mark.gpu
def test_suite_records_every_format(tmp_path):
    """sizes {50, 129}: 6 full + 4 packed + 12 RFP records per size (packed
    has no inverse), every residual within the tolerance, positive finite
    Mflop/s, and a second run with the same seed reproduces every non-timing
    field."""
    recs = B.run_suite([50, 129], reps=3, seed=11, nrhs=17)
    assert len(recs) == 2 * (6 + 4 + 12)
    for r in recs:
        assert not r.failed and r.residual <= 10.0
        assert math.isfinite(r.mflops) and r.mflops > 0
        assert (r.transr in "NT" and r.transr) if r.format == "rfp" else r.transr == ""
        assert r.nrhs == (17 if r.routine == "solve" else 0)
    again = B.run_suite([50, 129], reps=3, seed=11, nrhs=17)
    key = lambda r: (r.routine, r.format, r.n, r.nrhs, r.uplo, r.transr, r.reps, r.residual,
                     r.seed)
    assert [key(r) for r in recs] == [key(r) for r in again]
    p = tmp_path / "suite.csv"
    assert B.main(["--sizes", "64", "--reps", "3", "--out", str(p)]) == 0
    back = B.read_csv(p)
    assert len(back) == 6 + 4 + 12 and os.path.getsize(p) > 0
