"""GPU parity of the full-format device kernels (kernels.py surface) against
the CPU oracle on random strided views: every side/uplo/trans/diag flag
combination, real and complex, column- and row-major operands."""

import itertools

import numpy as np
import pytest
import torch

from oracle import rfp_oracle as O

pytestmark = pytest.mark.gpu
TOL = 1e-10


def rel(a, b):
    a = a.cpu().numpy() if isinstance(a, torch.Tensor) else a
    return float(np.abs(a - b).max()) / max(float(np.abs(b).max()), 1e-300)


def rnd(shape, cplx, seed, rowmajor=False):
    g = np.random.default_rng(seed)
    x = g.standard_normal(shape) + (1j * g.standard_normal(shape) if cplx else 0)
    return np.ascontiguousarray(x) if rowmajor else np.asfortranarray(x)


def dev(x):
    t = torch.from_numpy(x).cuda()
    return t


def tri_matrix(n, cplx, seed, rowmajor):
    t = rnd((n, n), cplx, seed, rowmajor)
    t[np.diag_indices(n)] += 2 * n  # well conditioned triangles
    return t


@pytest.fixture(scope="module")
def K():
    from paper_0901_1696_b200 import kernels
    return kernels


@pytest.mark.parametrize("cplx", [False, True])
@pytest.mark.parametrize("ta,tb", list(itertools.product("NTC", "NTC")))
@pytest.mark.parametrize("m,n,k", [(70, 45, 33), (200, 130, 257)])
def test_gemm(K, cplx, ta, tb, m, n, k):
    a = rnd((m, k) if ta == "N" else (k, m), cplx, 1, rowmajor=(m % 2 == 0))
    b = rnd((k, n) if tb == "N" else (n, k), cplx, 2)
    c = rnd((m, n), cplx, 3, rowmajor=(k % 2 == 1))
    want = c.copy()
    O.gemm(ta, tb, -1.0, a, b, 0.5, want)
    cd = dev(c)
    K.gemm(ta, tb, -1.0, dev(a), dev(b), 0.5, cd)
    assert rel(cd, want) <= TOL


@pytest.mark.parametrize("cplx", [False, True])
@pytest.mark.parametrize("side,uplo,trans,diag", list(itertools.product("LR", "LU", "NTC", "NU")))
def test_trsm_trmm(K, cplx, side, uplo, trans, diag):
    n, r = 150, 37
    a = tri_matrix(n, cplx, 5, rowmajor=(uplo == "U"))
    b = rnd((n, r) if side == "L" else (r, n), cplx, 6, rowmajor=(trans == "T"))
    want = b.copy()
    O.trsm(side, uplo, trans, diag, 2.0, a, want)
    bd = dev(b)
    K.trsm(side, uplo, trans, diag, 2.0, dev(a), bd)
    assert rel(bd, want) <= TOL
    want = b.copy()
    O.trmm(side, uplo, trans, diag, -1.5, a, want)
    bd = dev(b)
    K.trmm(side, uplo, trans, diag, -1.5, dev(a), bd)
    assert rel(bd, want) <= TOL


def test_trsm_singular(K):
    a = tri_matrix(80, False, 1, False)
    a[70, 70] = 0.0
    a[10, 10] = 0.0
    with pytest.raises(K.SingularMatrixError) as e:
        K.trsm("L", "L", "N", "N", 1.0, dev(a), dev(rnd((80, 3), False, 2)))
    assert e.value.index == 11
    with pytest.raises(K.SingularMatrixError) as e:
        K.trsm("L", "U", "N", "N", 1.0, dev(a), dev(rnd((80, 3), False, 2)))
    assert e.value.index == 71


@pytest.mark.parametrize("cplx", [False, True])
@pytest.mark.parametrize("uplo,trans", list(itertools.product("LU", "NTC")))
def test_syrk_herk(K, cplx, uplo, trans):
    n, k = 190, 77
    a = rnd((n, k) if trans == "N" else (k, n), cplx, 7)
    c = rnd((n, n), cplx, 8, rowmajor=(uplo == "L"))
    for herm in ([False, True] if cplx else [False]):
        want = c.copy()
        O.syrk_herk(uplo, trans, -1.0, a, 1.0, want, herm)
        cd = dev(c)
        K.syrk_herk(uplo, trans, -1.0, dev(a), 1.0, cd, hermitian=herm)
        assert rel(cd, want) <= TOL
        # the other triangle is bit-identical
        other = np.triu(np.ones((n, n), bool), 1) if uplo == "L" else np.tril(np.ones((n, n), bool), -1)
        assert np.array_equal(cd.cpu().numpy()[other], c[other])


@pytest.mark.parametrize("cplx", [False, True])
@pytest.mark.parametrize("uplo", "LU")
@pytest.mark.parametrize("n", [1, 50, 64, 65, 200, 333])
def test_potrf_trtri_lauum(K, cplx, uplo, n):
    g = rnd((n, n), cplx, n)
    a = np.asfortranarray(g @ np.conj(g.T) + n * np.eye(n))
    want = a.copy(order="F")
    assert O.potrf(uplo, want) == 0
    ad = dev(a)
    assert K.potrf_ref(uplo, ad) == 0
    assert rel(ad, want) <= TOL
    other = np.triu(np.ones((n, n), bool), 1) if uplo == "L" else np.tril(np.ones((n, n), bool), -1)
    assert np.array_equal(ad.cpu().numpy()[other], a[other])
    for diag in "NU":
        w2 = want.copy(order="F")
        assert O.trtri(uplo, diag, w2) == 0
        td = dev(want.copy(order="F"))
        assert K.trtri_ref(uplo, diag, td) == 0
        assert rel(td, w2) <= TOL
    w3 = want.copy(order="F")
    O.lauum(uplo, w3)
    ld = dev(want.copy(order="F"))
    K.lauum_ref(uplo, ld)
    assert rel(ld, w3) <= TOL


def test_potrf_failure_and_trtri_zero(K):
    n = 150
    a = np.eye(n) * 4.0
    a[120, 120] = -1.0
    ad = dev(np.asfortranarray(a))
    assert K.potrf_ref("L", ad) == O.potrf("L", a.copy()) == 121
    t = np.asfortranarray(np.tril(rnd((n, n), False, 3)) + 10 * np.eye(n))
    t[77, 77] = 0.0
    td = dev(t)
    assert K.trtri_ref("L", "N", td) == 78
    assert np.array_equal(td.cpu().numpy(), t)  # untouched (kernels.py:526-529)


@pytest.mark.parametrize("uplo", "LU")
def test_zpotrf_split_level(K, uplo):
    """Complex potrf with the GEMM-level split forced at a small order (tuning
    zpotrf_split_min): the halves on the tile kernel, the panel solve and the
    HERK between them; the factor against the oracle, and a failing pivot in
    each half reported at its global index."""
    from paper_0901_1696_b200 import _capi
    n = 700
    g = rnd((n, n), True, 31)
    a = np.asfortranarray(g @ np.conj(g.T) + n * np.eye(n))
    want = a.copy(order="F")
    assert O.potrf(uplo, want) == 0
    with _capi.tuning(zpotrf_split_min=300):
        ad = dev(a)
        assert K.potrf_ref(uplo, ad) == 0
        assert rel(ad, want) <= TOL
        for bad in (100, 500):
            b = a.copy(order="F")
            b[bad, bad] = -1.0
            assert K.potrf_ref(uplo, dev(b)) == O.potrf(uplo, b.copy(order="F")) == bad + 1


# ---------------------------------------------------------------- dataflow tile kernels
@pytest.mark.parametrize("cplx", [False, True])
@pytest.mark.parametrize("uplo", "LU")
def test_tile_kernels_repeat_stress(K, cplx, uplo):
    """The persistent tile potrf / trsm kernels synchronise through device
    flags; run every tile-count regime (1, 2, 3, many tiles; partial last
    tile) several times against torch's cuSOLVER/cuBLAS in FP64, so an
    ordering race would show up as a mismatch or a varying result."""
    for n in (64, 65, 128, 130, 200, 700, 1500):
        g = np.random.default_rng(n)
        b = g.standard_normal((n, n)) + (1j * g.standard_normal((n, n)) if cplx else 0)
        a = b @ b.conj().T / n + np.eye(n)
        ref = np.linalg.cholesky(a)
        want = ref if uplo == "L" else ref.conj().T
        rhs = g.standard_normal((n, 70)) + (1j * g.standard_normal((n, 70)) if cplx else 0)
        xs = np.linalg.solve(ref, rhs)
        first = None
        for rep in range(3):
            ad = dev(np.asfortranarray(a.copy()))
            assert K.potrf_ref(uplo, ad) == 0
            got = ad.cpu().numpy()
            got = np.tril(got) if uplo == "L" else np.triu(got)
            assert rel(got, want) <= 1e-10, (n, rep)
            if first is None:
                first = got
            else:
                assert np.array_equal(got, first), (n, rep)  # deterministic
            bd = dev(np.asfortranarray(rhs.copy()))
            lo = dev(np.asfortranarray(ref.copy()))
            K.trsm("L", "L", "N", "N", 1.0, lo, bd)
            assert rel(bd, xs) <= 1e-10, (n, rep)
            if rep == 0:
                first_x = bd.cpu().numpy()
            else:
                assert np.array_equal(bd.cpu().numpy(), first_x), (n, rep)  # deterministic


@pytest.mark.parametrize("side,uplo,trans", list(itertools.product("LR", "LU", "NT")))
@pytest.mark.parametrize("r", [1, 37, 64, 200, 300])
def test_tile_trsm_widths(K, side, uplo, trans, r):
    """The dataflow trsm (n >= 512) in both tile widths: 64 x 16 tiles for
    narrow right-hand sides (r <= 256) and 64 x 64 above; ragged last tiles
    in both dimensions (n = 600), column- and row-major B."""
    n = 600
    a = tri_matrix(n, False, 11, rowmajor=(uplo == "U"))
    b = rnd((n, r) if side == "L" else (r, n), False, 12 + r, rowmajor=(trans == "T"))
    want = b.copy()
    O.trsm(side, uplo, trans, "N", 1.5, a, want)
    bd = dev(b)
    K.trsm(side, uplo, trans, "N", 1.5, dev(a), bd)
    assert rel(bd, want) <= TOL


@pytest.mark.parametrize("side,uplo,trans", [("L", "L", "N"), ("L", "L", "T"), ("L", "U", "N"),
                                             ("L", "U", "T"), ("R", "L", "T"), ("R", "U", "N")])
def test_tile_trsm_split_tasks(K, side, uplo, trans):
    """Split tasks of the wide-tile dataflow trsm (tuning trsm_split): from
    solve position 6 on, a PRE task sums all but the last 3 chunks of every
    tile and updates B in place, the tile's own task waits for it.  Ragged
    last tiles in both dimensions, forward and backward sweeps, against the
    oracle and against the unsplit solve."""
    from paper_0901_1696_b200 import _capi
    n, r = 1800, 4000
    a = tri_matrix(n, False, 21, rowmajor=(uplo == "U"))
    b = rnd((n, r) if side == "L" else (r, n), False, 22, rowmajor=(side == "R"))
    want = b.copy()
    O.trsm(side, uplo, trans, "N", 1.0, a, want)
    got = {}
    for split in (0, 3):
        with _capi.tuning(trsm_split=split):
            bd = dev(b)
            K.trsm(side, uplo, trans, "N", 1.0, dev(a), bd)
            got[split] = bd.cpu().numpy()
            assert rel(got[split], want) <= TOL, split
    assert not np.array_equal(got[0], got[3])  # the split path ran (other summation order)


@pytest.mark.parametrize("cplx", [False, True])
def test_gemm_splitk_deterministic(K, cplx):
    """Few output tiles and a long K take the split-K path (partials reduced
    in a fixed order): results match the oracle and repeat bit for bit."""
    m, n, k = 300, 64, 3000
    a = rnd((m, k), cplx, 21)
    b = rnd((k, n), cplx, 22)
    c = rnd((m, n), cplx, 23)
    want = c.copy()
    O.gemm("N", "N", -1.0, a, b, 0.5, want)
    outs = []
    for _ in range(3):
        cd = dev(c)
        K.gemm("N", "N", -1.0, dev(a), dev(b), 0.5, cd)
        outs.append(cd.cpu().numpy())
    assert rel(outs[0], want) <= TOL
    assert all(np.array_equal(o, outs[0]) for o in outs[1:])


def test_gemm_wide_tiles(K):
    """Large outputs take the 64 x 128 tile configuration (>= 4 waves of
    tiles); ragged edges in both dimensions."""
    m, n, k = 4096 + 17, 4096 + 33, 40
    a = rnd((m, k), False, 31)
    b = rnd((n, k), False, 32)
    c = rnd((m, n), False, 33)
    want = c.copy()
    O.gemm("N", "T", 1.5, a, b, -0.5, want)
    cd = dev(c)
    K.gemm("N", "T", 1.5, dev(a), dev(b), -0.5, cd)
    assert rel(cd, want) <= TOL


@pytest.mark.parametrize("uplo,trans", [("L", "N"), ("U", "N"), ("L", "T"), ("U", "T")])
def test_syrk_large(K, uplo, trans):
    """SYRK over many triangular tiles with ragged edges: exactly the declared
    triangle is updated (the other one stays bit-identical)."""
    n, k = 4700, 24
    a = rnd((n, k) if trans == "N" else (k, n), False, 34)
    c = rnd((n, n), False, 35, rowmajor=(uplo == "U"))
    want = c.copy()
    O.syrk_herk(uplo, trans, -1.0, a, 1.0, want, False)
    cd = dev(c)
    K.syrk_herk(uplo, trans, -1.0, dev(a), 1.0, cd, hermitian=False)
    assert rel(cd, want) <= TOL
    other = np.triu(np.ones((n, n), bool), 1) if uplo == "L" else np.tril(np.ones((n, n), bool), -1)
    assert np.array_equal(cd.cpu().numpy()[other], c[other])


def test_forced_wide_tiles_triangular(K):
    """Tuning gemm_wide=1 forces the 64 x 128 tiles onto SYRK too (the
    non-square triangular tile enumeration): other triangle untouched,
    values against the oracle."""
    from paper_0901_1696_b200 import _capi
    with _capi.tuning(gemm_wide=1):
        for uplo in "LU":
            g = np.random.default_rng(5)
            a = np.asfortranarray(g.standard_normal((700, 19)))
            c = np.asfortranarray(g.standard_normal((700, 700)))
            want = c.copy()
            O.syrk_herk(uplo, "N", -1.0, a, 1.0, want, False)
            cd = torch.from_numpy(c).cuda()
            K.syrk_herk(uplo, "N", -1.0, torch.from_numpy(a).cuda(), 1.0, cd)
            got = cd.cpu().numpy()
            assert np.abs(got - want).max() <= TOL * np.abs(want).max(), uplo
            other = (np.triu(np.ones((700, 700), bool), 1) if uplo == "L"
                     else np.tril(np.ones((700, 700), bool), -1))
            assert np.array_equal(got[other], c[other]), uplo


@pytest.mark.parametrize("cplx", [False, True])
@pytest.mark.parametrize("diag", "NU")
def test_trtri_hybrid_large(K, cplx, diag):
    """Orders above the one-launch size (4096) run the hybrid recursion (top
    trmm levels, sub-blocks <= 4096 on the tile trsm); checked against torch's
    FP64 triangular solve with the identity."""
    n = 4500
    g = torch.Generator(device="cuda").manual_seed(7)
    dt = torch.complex128 if cplx else torch.float64
    a = torch.randn(n, n, dtype=dt, device="cuda", generator=g)
    # unit diagonal: small off-diagonal entries keep L^-1 bounded (with N(0,1)
    # entries a unit triangle's inverse grows exponentially and overflows)
    scale = 1.0 / (2 * n) if diag == "U" else 1.0
    a = torch.triu(a) + scale * torch.tril(a, -1) + 2 * n * torch.eye(n, dtype=dt, device="cuda")
    want_l = torch.tril(a)
    if diag == "U":
        want_l = want_l - torch.diag(torch.diagonal(want_l)) + torch.eye(n, dtype=dt, device="cuda")
    want = torch.linalg.solve_triangular(want_l, torch.eye(n, dtype=dt, device="cuda"), upper=False)
    got = a.clone()
    assert K.trtri_ref("L", diag, got) == 0
    low = torch.tril(torch.ones(n, n, dtype=torch.bool, device="cuda"), -1 if diag == "U" else 0)
    err = (got - want)[low].abs().max() / want[low].abs().max()
    assert float(err) <= TOL
    if diag == "U":  # the stored diagonal is never referenced nor written
        assert torch.equal(torch.diagonal(got), torch.diagonal(a))
    assert torch.equal(torch.triu(got, 1), torch.triu(a, 1))
