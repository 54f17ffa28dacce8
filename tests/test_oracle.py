"""Pin the CPU oracle to the reference: golden vectors produced by the
reference itself (tests/golden/make_golden.py), SPEC.md known answers and
the layout doctests; plus scipy's LAPACK RFP routines as a second oracle."""

import numpy as np
import pytest

from oracle import rfp_oracle as O
from tests.conftest import golden_cases


def _cases():
    with np.load(__import__("tests.conftest", fromlist=["GOLDEN"]).GOLDEN) as z:
        return golden_cases({k: None for k in z.files})


CASES = _cases()


def rel(a, b):
    den = max(float(np.abs(b).max()), 1e-300) if b.size else 1.0
    return float(np.abs(a - b).max()) / den if a.size else 0.0


@pytest.mark.parametrize("key,dt,uplo,transr,n", CASES, ids=[c[0] for c in CASES])
def test_conversions_bit_exact(golden, key, dt, uplo, transr, n):
    a = golden[key + "_A"]
    buf = O.trttf(a, uplo, transr)
    assert buf.tobytes() == golden[key + "_rfp"].tobytes()
    assert O.tfttr(buf, n, uplo, transr).tobytes() == golden[key + "_tfttr"].tobytes()
    p = O.pack(a, uplo)
    assert p.tobytes() == golden[key + "_packed"].tobytes()
    assert O.tpttf(p, n, uplo, transr).tobytes() == golden[key + "_tpttf"].tobytes()
    assert O.tfttp(buf, n, uplo, transr).tobytes() == golden[key + "_tfttp"].tobytes()


@pytest.mark.parametrize("key,dt,uplo,transr,n", CASES, ids=[c[0] for c in CASES])
def test_compute_matches_reference(golden, key, dt, uplo, transr, n):
    f = golden[key + "_rfp"].copy()
    assert O.pftrf(f, n, uplo, transr) == int(golden[key + "_pftrf_info"])
    assert rel(f, golden[key + "_factor"]) <= 1e-13
    x = golden[key + "_B"].copy(order="F")
    O.pftrs(golden[key + "_factor"], n, uplo, transr, x)
    assert rel(x, golden[key + "_X"]) <= 1e-13
    t = golden[key + "_factor"].copy()
    assert O.tftri(t, n, uplo, transr) == int(golden[key + "_tftri_info"])
    assert rel(t, golden[key + "_tftri"]) <= 1e-13
    inv = golden[key + "_factor"].copy()
    assert O.pftri(inv, n, uplo, transr) == int(golden[key + "_pftri_info"])
    assert rel(inv, golden[key + "_pftri"]) <= 1e-13


def test_failure_indices(golden):
    keys = [k[:-5] for k in golden if k.startswith("fail_") and k.endswith("_info")]
    assert len(keys) >= 50
    for base in keys:
        _, dt, ut, nn, *_ = base.split("_")
        buf = golden[base + "_rfp"].copy()
        assert O.pftrf(buf, int(nn[1:]), ut[0], ut[1]) == int(golden[base + "_info"]), base


def test_spec_known_answers(golden):
    # n=2 [[4,.],[2,5]] factors to [[2,.],[1,2]]; buffer [5,4,2] -> [2,2,1]
    buf = O.trttf(np.array([[4.0, 0.0], [2.0, 5.0]]), "L", "N")
    assert buf.tolist() == [5.0, 4.0, 2.0] == golden["spec_n2_rfp"].tolist()
    assert O.pftrf(buf, 2, "L", "N") == 0
    assert buf.tolist() == [2.0, 2.0, 1.0] == golden["spec_n2_factor"].tolist()
    # inverse [[5/16,.],[-1/8,1/4]]
    assert O.pftri(buf, 2, "L", "N") == 0
    full = O.tfttr(buf, 2, "L", "N")
    assert np.array_equal(full, np.array([[0.3125, 0.0], [-0.125, 0.25]]))
    assert np.array_equal(full, golden["spec_n2_inverse_full"])
    # non-PD [[1,.],[2,1]] -> info 2
    bad = O.trttf(np.array([[1.0, 0.0], [2.0, 1.0]]), "L", "N")
    assert O.pftrf(bad, 2, "L", "N") == 2 == int(golden["spec_n2_bad_info"])


def test_layout_known_answers():
    from paper_0901_1696_b200 import layout as L
    d = L.make_descriptor(7, "L", "N")
    assert (d.n1, d.n2, d.nt, d.ldar) == (4, 3, 28, 7)
    assert [L.map_index(d, 5, 5), L.map_index(d, 7, 4), L.map_index(d, 2, 1)] == [8, 28, 2]
    d6 = L.make_descriptor(6, "L", "N")
    assert (d6.n1, d6.n2, d6.nt, d6.ldar) == (3, 3, 21, 7)
    assert [L.map_index(d6, 4, 4), L.map_index(d6, 6, 4), L.map_index(d6, 6, 5)] == [1, 15, 16]
    u6 = L.make_descriptor(6, "U", "N")
    assert [L.map_index(u6, 4, 5), L.map_index(u6, 5, 6)] == [11, 19]
    d1 = L.make_descriptor(1, "U", "T")
    assert (d1.n1, d1.n2, d1.nt, d1.ldar) == (1, 0, 1, 1)
    assert L.make_descriptor(5, "lower", "C").transr == "T"
    with pytest.raises(ValueError):
        L.make_descriptor(3, "X", "N")
    with pytest.raises(ValueError):
        L.make_descriptor(-1, "L", "N")
    with pytest.raises(IndexError):
        L.map_index(d, 1, 2)


@pytest.mark.parametrize("uplo", "LU")
@pytest.mark.parametrize("transr", "NT")
@pytest.mark.parametrize("n", range(0, 41))
def test_map_index_bijective_and_matches_oracle(uplo, transr, n):
    from paper_0901_1696_b200 import layout as L
    d = L.make_descriptor(n, uplo, transr)
    seen = set()
    a = np.arange(1, n * n + 1, dtype=np.float64).reshape(n, n, order="F")
    buf = O.trttf(a, uplo, transr)
    for j in range(1, n + 1):
        for i in (range(j, n + 1) if uplo == "L" else range(1, j + 1)):
            off = L.map_index(d, i, j)
            seen.add(off)
            assert buf[off - 1] == a[i - 1, j - 1]
    assert seen == set(range(1, d.nt + 1))


def test_block_geometry_matches_oracle_views():
    from paper_0901_1696_b200 import layout as L
    for n in (1, 2, 5, 6, 40, 41):
        for uplo in "LU":
            for transr in "NT":
                d = L.make_descriptor(n, uplo, transr)
                buf = np.arange(d.nt, dtype=np.float64)
                views = O.blocks(buf, O.desc(n, uplo, transr))
                for (off, rows, cols, rs, cs), v in zip(L.block_geometry(d), views):
                    assert v.shape == (rows, cols)
                    if v.size:
                        ii, jj = np.meshgrid(np.arange(rows), np.arange(cols), indexing="ij")
                        assert np.array_equal(v, buf[off + ii * rs + jj * cs])


@pytest.mark.parametrize("n", [1, 2, 6, 7, 40, 41])
@pytest.mark.parametrize("uplo", "LU")
@pytest.mark.parametrize("transr", "NT")
def test_scipy_lapack_second_oracle(n, uplo, transr):
    """Real RFP buffers are bit-identical to LAPACK dtrttf; factors, solves
    and inverses agree to rounding."""
    from scipy.linalg import lapack
    a = O.spd_matrix(n, 5 + n, "n")
    buf = O.trttf(a, uplo, transr)
    arf, info = lapack.dtrttf(a, transr=transr, uplo=uplo)
    assert info == 0 and arf.tobytes() == buf.tobytes()
    f = buf.copy()
    assert O.pftrf(f, n, uplo, transr) == 0
    lf, info = lapack.dpftrf(n, arf, transr=transr, uplo=uplo)
    assert info == 0 and rel(f, lf) <= 1e-13
    b = np.asfortranarray(np.random.default_rng(n).standard_normal((n, 4)))
    x = b.copy(order="F")
    O.pftrs(f, n, uplo, transr, x)
    lx, info = lapack.dpftrs(n, lf, b, transr=transr, uplo=uplo)
    assert rel(x, lx) <= 1e-12
    inv = f.copy()
    O.pftri(inv, n, uplo, transr)
    li, info = lapack.dpftri(n, lf, transr=transr, uplo=uplo)
    assert rel(inv, li) <= 1e-12


# ---------------------------------------------------------------- SURVEY 8(f) rows
from tests.conftest import next_row_cases  # noqa: E402

with np.load(__import__("tests.conftest", fromlist=["GOLDEN"]).GOLDEN) as _z:
    NEXT = next_row_cases({k: None for k in _z.files})


@pytest.mark.parametrize("key,dt,uplo,transr,n", NEXT, ids=[c[0] for c in NEXT])
def test_next_rows_match_reference(golden, key, dt, uplo, transr, n):
    f = golden[f"tfsm_{key}_factor"]
    cplx = dt == "c128"
    for side in "LR":
        for trans in "NTC":
            for diag in "NU":
                b = golden[f"tfsm_{key}_{side}{trans}{diag}_B"].copy(order="F")
                alpha = (1.5 - 0.5j) if cplx else 1.5
                O.tfsm(f, n, uplo, transr, side, trans, diag, alpha, b)
                assert rel(b, golden[f"tfsm_{key}_{side}{trans}{diag}_X"]) <= 1e-12, (side, trans, diag)
    for trans in "NC":
        c = golden[f"sfrk_{key}_{trans}_C0"].copy()
        O.sfrk_hfrk(c, n, uplo, transr, trans, 5, -0.75, golden[f"sfrk_{key}_{trans}_A"], 1.25, cplx)
        assert rel(c, golden[f"sfrk_{key}_{trans}_C"]) <= 1e-13
    want = golden[f"lansf_{key}"]
    got = [O.lansf(nm, golden[f"lansf_{key}_rfp"], n, uplo, transr) for nm in "M1IF"]
    assert np.allclose(got, want, rtol=1e-13, atol=0)


# ---------------------------------------------------------------- SURVEY 8(f) row 4
def _pp_keys(g):
    return sorted(k[:-len("_info")] for k in g if k.startswith("pp_") and k.endswith("_info"))


def test_packed_cholesky_matches_reference(golden):
    keys = _pp_keys(golden)
    assert len(keys) >= 30
    for key in keys:
        _, dt, uplo, nn, *rest = key.split("_")
        n = int(nn[1:])
        p = golden[key + "_P"].copy()
        assert O.pptrf(p, n, uplo) == int(golden[key + "_info"]), key
        if rest:  # failing case: only the index is specified
            continue
        assert rel(p, golden[key + "_F"]) <= 1e-13, key
        x = golden[key + "_B"].copy(order="F")
        O.pptrs(golden[key + "_F"], n, uplo, x)
        assert rel(x, golden[key + "_X"]) <= 1e-13, key
