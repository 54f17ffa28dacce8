"""GPU parity: the sm_100a path (through the C ABI) against the reference's
golden vectors and the CPU oracle.  Conversions must be bit-exact; factors,
solutions and inverses within 1e-10 max-relative of the oracle
(BASELINE.json north_star tolerance); info codes identical."""

import numpy as np
import pytest
import torch

from oracle import rfp_oracle as O
from tests.conftest import golden_cases, GOLDEN

pytestmark = pytest.mark.gpu

with np.load(GOLDEN) as _z:
    CASES = golden_cases({k: None for k in _z.files})

TOL = 1e-10


def rel(a, b):
    a = a.cpu().numpy() if isinstance(a, torch.Tensor) else np.asarray(a)
    b = b.cpu().numpy() if isinstance(b, torch.Tensor) else np.asarray(b)
    if a.size == 0:
        return 0.0
    return float(np.abs(a - b).max()) / max(float(np.abs(b).max()), 1e-300)


def bits(t):
    return t.detach().cpu().numpy().tobytes()


@pytest.fixture(scope="module")
def P():
    import paper_0901_1696_b200 as pkg
    from paper_0901_1696_b200 import convert, packed, rfp, kernels  # noqa: F401
    assert torch.cuda.is_available()
    return pkg


@pytest.mark.parametrize("key,dt,uplo,transr,n", CASES, ids=[c[0] for c in CASES])
def test_conversions_bit_exact(P, golden, key, dt, uplo, transr, n):
    conv, packed = P.convert, P.packed
    a = golden[key + "_A"]
    r = conv.trttf(a, uplo, transr)
    assert r.data.is_cuda
    assert bits(r.data) == golden[key + "_rfp"].tobytes()
    full = conv.tfttr(r)
    assert full.stride(0) == 1 or n <= 1
    assert bits(full.t().contiguous().t()) == np.asfortranarray(golden[key + "_tfttr"]).tobytes()
    full7 = conv.tfttr(r, ld=n + 7)
    assert full7.shape == (n + 7, n) and float(full7[n:].abs().sum()) == 0.0
    p = packed.pack(a, uplo)
    assert bits(p.data) == golden[key + "_packed"].tobytes()
    assert bits(conv.tpttf(p, transr).data) == golden[key + "_tpttf"].tobytes()
    assert bits(conv.tfttp(r).data) == golden[key + "_tfttp"].tobytes()
    back = packed.unpack(p)
    assert bits(back.t().contiguous().t()) == np.asfortranarray(golden[key + "_tfttr"]).tobytes()


@pytest.mark.parametrize("key,dt,uplo,transr,n", CASES, ids=[c[0] for c in CASES])
def test_pftrf_pftrs_pftri_match_reference(P, golden, key, dt, uplo, transr, n):
    conv, rfp, layout = P.convert, P.rfp, P.layout
    d = layout.make_descriptor(n, uplo, transr)
    r = conv.RfpTriangle(golden[key + "_rfp"], d)
    assert rfp.pftrf(r) == int(golden[key + "_pftrf_info"])
    assert r.state is conv.FactorState.CHOLESKY
    assert rel(r.data, golden[key + "_factor"]) <= TOL
    b = torch.from_numpy(golden[key + "_B"]).cuda()
    x = b.clone()
    rfp.pftrs(r, x)
    assert rel(x, golden[key + "_X"]) <= TOL
    # row-major RHS and 1-D RHS
    xr = torch.from_numpy(np.ascontiguousarray(golden[key + "_B"])).cuda()
    rfp.pftrs(r, xr)
    assert rel(xr, golden[key + "_X"]) <= TOL
    if n:
        x1 = torch.from_numpy(golden[key + "_B"][:, 0].copy()).cuda()
        rfp.pftrs(r, x1)
        assert rel(x1, golden[key + "_X"][:, 0]) <= TOL
    t = r.copy()
    assert rfp.tftri(t) == int(golden[key + "_tftri_info"])
    assert rel(t.data, golden[key + "_tftri"]) <= TOL
    inv = r.copy()
    assert rfp.pftri(inv) == int(golden[key + "_pftri_info"])
    assert inv.state is conv.FactorState.FULL_INVERSE
    assert rel(inv.data, golden[key + "_pftri"]) <= TOL


def test_failure_info_matches_reference(P, golden):
    conv, rfp, layout = P.convert, P.rfp, P.layout
    keys = [k[:-5] for k in golden if k.startswith("fail_") and k.endswith("_info")]
    for base in keys:
        _, dt, ut, nn, *_ = base.split("_")
        n = int(nn[1:])
        r = conv.RfpTriangle(golden[base + "_rfp"], layout.make_descriptor(n, ut[0], ut[1]))
        assert rfp.pftrf(r) == int(golden[base + "_info"]), base
        assert r.state is conv.FactorState.UNFACTORED


def test_state_machine_and_errors(P):
    conv, rfp, layout = P.convert, P.rfp, P.layout
    r = conv.trttf(O.spd_matrix(5, 1), "L", "N")
    with pytest.raises(ValueError, match="pftrs needs a Cholesky factor"):
        rfp.pftrs(r, torch.zeros(5, 1, dtype=torch.float64, device="cuda"))
    with pytest.raises(ValueError, match="pftri needs a Cholesky factor"):
        rfp.pftri(r)
    assert rfp.pftrf(r) == 0
    with pytest.raises(ValueError, match="does not match order"):
        rfp.pftrs(r, torch.zeros(4, 1, dtype=torch.float64, device="cuda"))
    z = conv.trttf(O.spd_matrix(5, 2, complex_=True), "U", "C")
    assert z.desc.transr == "T"
    assert rfp.pftrf(z) == 0
    with pytest.raises(ValueError, match="complex system"):
        rfp.pftrs(z, torch.zeros(5, 1, dtype=torch.float64, device="cuda"))
    e = conv.RfpTriangle(torch.zeros(0, dtype=torch.float64), layout.make_descriptor(0, "L", "N"))
    assert rfp.pftrf(e) == 0 and e.state is conv.FactorState.CHOLESKY
    assert rfp.pftri(e) == 0 and e.state is conv.FactorState.FULL_INVERSE
    with pytest.raises(ValueError):
        conv.RfpTriangle(torch.zeros(7, dtype=torch.float64), layout.make_descriptor(3, "L", "N"))


def test_host_rhs_is_solved_in_place(P):
    conv, rfp = P.convert, P.rfp
    a = O.spd_matrix(9, 3)
    r = conv.trttf(a, "U", "T")
    assert rfp.pftrf(r) == 0
    b = np.asfortranarray(np.random.default_rng(0).standard_normal((9, 2)))
    x = b.copy(order="F")
    rfp.pftrs(r, x)
    assert np.abs(a @ x - b).max() < 1e-12
    # real factor with complex RHS (rfp.py:101 allows it)
    bc = torch.from_numpy(b + 1j * b[::-1]).cuda()
    xc = bc.clone()
    rfp.pftrs(r, xc)
    ac = torch.from_numpy(a).cuda().to(torch.complex128)
    assert float((ac @ xc - bc).abs().max()) < 1e-12


@pytest.mark.parametrize("n", [65, 128, 130, 257, 600])
@pytest.mark.parametrize("uplo,transr", [("L", "N"), ("U", "T"), ("L", "T"), ("U", "N")])
@pytest.mark.parametrize("cplx", [False, True])
def test_recursive_sizes_vs_oracle(P, n, uplo, transr, cplx):
    """Sizes beyond the 64 leaf exercise the recursive drivers and GEMMs."""
    conv, rfp = P.convert, P.rfp
    a = O.spd_matrix(n, 100 + n, "n", complex_=cplx)
    buf = O.trttf(a, uplo, transr)
    f = buf.copy()
    assert O.pftrf(f, n, uplo, transr) == 0
    r = conv.trttf(a, uplo, transr)
    assert bits(r.data) == buf.tobytes()
    assert rfp.pftrf(r) == 0
    assert rel(r.data, f) <= TOL
    rng = np.random.default_rng(n)
    b = rng.standard_normal((n, 7)) + (1j * rng.standard_normal((n, 7)) if cplx else 0)
    b = np.asfortranarray(b)
    xo = b.copy(order="F")
    O.pftrs(f, n, uplo, transr, xo)
    x = torch.from_numpy(b).cuda()
    rfp.pftrs(r, x)
    assert rel(x, xo) <= TOL
    inv_o = f.copy()
    O.pftri(inv_o, n, uplo, transr)
    assert rfp.pftri(r) == 0
    assert rel(r.data, inv_o) <= TOL


def test_batched_vs_oracle(P):
    rfp = P.rfp
    for n, uplo, transr, nrhs in [(64, "U", "N", 8), (64, "L", "T", 3), (33, "L", "N", 1),
                                  (1, "U", "T", 2), (17, "U", "C", 8), (64, "L", "N", 0),
                                  (64, "L", "N", 13), (64, "U", "T", 8), (64, "U", "C", 1),
                                  (63, "U", "N", 8)]:
        batch = 37
        bufs, facs, xs, bs = [], [], [], []
        for k in range(batch):
            a = O.spd_matrix(n, 1000 + k, "n")
            buf = O.trttf(a, uplo, transr)
            bufs.append(buf)
            f = buf.copy()
            assert O.pftrf(f, n, uplo, transr) == 0
            facs.append(f)
            b = np.asfortranarray(np.random.default_rng(k).standard_normal((n, max(nrhs, 1))))
            bs.append(b)
            x = b.copy(order="F")
            O.pftrs(f, n, uplo, transr, x)
            xs.append(x)
        arf = torch.from_numpy(np.stack(bufs)).cuda()
        arf2 = arf.clone()
        bt = torch.from_numpy(np.stack([b.T for b in bs])).cuda().transpose(1, 2)[:, :, :nrhs]
        info = rfp.pftrf_pftrs_batched(arf, transr, uplo, n, bt)
        assert int(info.abs().sum()) == 0
        assert rel(arf, np.stack(facs)) <= TOL
        if nrhs:
            assert rel(bt, np.stack(xs)[:, :, :nrhs]) <= TOL
        # unfused
        info2 = rfp.pftrf_batched(arf2, transr, uplo, n)
        assert int(info2.abs().sum()) == 0
        assert rel(arf2, np.stack(facs)) <= TOL
        if nrhs:
            b2 = torch.from_numpy(np.stack(bs)).cuda()[:, :, :nrhs].contiguous()
            rfp.pftrs_batched(arf2, transr, uplo, n, b2)
            assert rel(b2, np.stack(xs)[:, :, :nrhs]) <= TOL


@pytest.mark.parametrize("uplo,transr", [("U", "N"), ("L", "N"), ("U", "T"), ("L", "T")])
def test_batched_failure_info(P, uplo, transr):
    rfp = P.rfp
    n, batch = 64, 8
    bufs, want = [], []
    for k in range(batch):
        a = O.spd_matrix(n, k, "n")
        if k % 3:
            # a non-PD pivot in the first (T1) or the second (T2) half
            p = k + 5 if k % 3 == 1 else 33 + k
            a[:, p] = 0.0
            a[p, :] = 0.0
            a[p, p] = -1.0
        buf = O.trttf(a, uplo, transr)
        want.append(O.pftrf(buf.copy(), n, uplo, transr))
        bufs.append(buf)
    arf = torch.from_numpy(np.stack(bufs)).cuda()
    info = rfp.pftrf_batched(arf, transr, uplo, n)
    assert info.cpu().tolist() == want
    assert any(0 < w <= 32 for w in want) and any(w > 32 for w in want)


def test_graph_replay_matches_direct(P):
    """Repeated calls on the same buffers are replayed from a cached CUDA
    graph (2nd call captures, 3rd+ replay); results must equal the first,
    directly launched, call bit for bit."""
    conv, rfp, layout = P.convert, P.rfp, P.layout
    from paper_0901_1696_b200 import _capi
    lib = _capi.lib()
    n = 700
    a = O.spd_matrix(n, 77, "n")
    src = conv.trttf(a, "U", "T")
    work = conv.RfpTriangle(src.data.clone(), src.desc)
    b0 = torch.from_numpy(np.asfortranarray(np.random.default_rng(5).standard_normal((n, 9)))).cuda()
    outs = []
    for rep in range(4):
        work.data.copy_(src.data)
        work.state = conv.FactorState.UNFACTORED
        assert rfp.pftrf(work) == 0
        x = b0.clone() if rep == 0 else x.copy_(b0)
        rfp.pftrs(work, x)
        outs.append((work.data.clone(), x.clone()))
    c0 = lib.rfpk_launch_count()
    work.data.copy_(src.data)
    work.state = conv.FactorState.UNFACTORED
    assert rfp.pftrf(work) == 0
    assert lib.rfpk_launch_count() > c0  # replayed kernels are counted
    for f, x in outs[1:]:
        assert torch.equal(f, outs[0][0]) and torch.equal(x, outs[0][1])


# ---------------------------------------------------------------- BASELINE configs


def _backward_error(P, buf_factor, a, n, uplo, transr):
    """||A - L L^H||_F / (n eps ||A||_F) with eps = 2^-53 (BASELINE.json)."""
    t = P.convert.tfttr(P.convert.RfpTriangle(buf_factor, P.layout.make_descriptor(n, uplo, transr)))
    f = t if uplo == "L" else t.mH
    r = a - f @ f.mH
    return float(torch.linalg.norm(r) / (n * 2.0 ** -53 * torch.linalg.norm(a)))


def test_config1_n1000_vs_oracle(P):
    """Config 1: n=1000 LN, A = B B^T + n I; pftrf, pftrs(100), pftri vs the oracle."""
    conv, rfp = P.convert, P.rfp
    n = 1000
    a = O.spd_matrix(n, 2024, "n")
    buf = O.trttf(a, "L", "N")
    r = conv.trttf(a, "L", "N")
    assert bits(r.data) == buf.tobytes()
    f = buf.copy()
    assert O.pftrf(f, n, "L", "N") == 0
    assert rfp.pftrf(r) == 0
    assert rel(r.data, f) <= TOL
    assert _backward_error(P, r.data, torch.from_numpy(a).cuda(), n, "L", "N") <= 10
    b = np.asfortranarray(np.random.default_rng(1).standard_normal((n, 100)))
    xo = b.copy(order="F")
    O.pftrs(f, n, "L", "N", xo)
    x = torch.from_numpy(b).cuda()
    rfp.pftrs(r, x)
    assert rel(x, xo) <= TOL
    O.pftri(f, n, "L", "N")
    assert rfp.pftri(r) == 0
    assert rel(r.data, f) <= TOL


@pytest.mark.parametrize("n", [4000, 4001])
@pytest.mark.parametrize("uplo", "LU")
@pytest.mark.parametrize("transr", "NT")
def test_config2_layout_sweep(P, n, uplo, transr):
    """Config 2: bit-exact trttf/tfttr and pack/tpttf/tfttp round trips at
    n = 4000/4001 in all 8 layouts (against the oracle's index maps), then
    pftrf (backward error <= 10) and pftrs(64) (scaled residual)."""
    conv, packed, rfp = P.convert, P.packed, P.rfp
    g = torch.Generator(device="cuda").manual_seed(n)
    bm = torch.randn(n, n, dtype=torch.float64, device="cuda", generator=g)
    a = bm @ bm.t()
    a.diagonal().add_(float(n))
    a = a.t().contiguous().t()
    r = conv.trttf(a, uplo, transr)
    ah = a.cpu().numpy()
    assert bits(r.data) == O.trttf(ah, uplo, transr).tobytes()
    full = conv.tfttr(r)
    want = torch.tril(a) if uplo == "L" else torch.triu(a)
    assert torch.equal(full, want)
    p = packed.pack(a, uplo)
    assert bits(p.data) == O.pack(ah, uplo).tobytes()
    r2 = conv.tpttf(p, transr)
    assert torch.equal(r2.data, r.data)
    assert torch.equal(conv.tfttp(r).data, p.data)
    assert rfp.pftrf(r) == 0
    assert _backward_error(P, r.data, a, n, uplo, transr) <= 10
    b = torch.randn(64, n, dtype=torch.float64, device="cuda", generator=g).t()
    x = b.clone()
    rfp.pftrs(r, x)
    res = float((a @ x - b).norm() / (a.norm() * x.norm() * n * 2.0 ** -53))
    assert res <= 10


def test_config3_n16384_properties(P):
    """Config 3 at full size: pftrf backward error <= 10 and pftrs(1024) residual."""
    conv, rfp = P.convert, P.rfp
    n, nrhs = 16384, 1024
    g = torch.Generator(device="cuda").manual_seed(3)
    bm = torch.randn(n, n, dtype=torch.float64, device="cuda", generator=g)
    a = bm @ bm.t()
    del bm
    a /= n
    a.diagonal().add_(1.0)
    r = conv.trttf(a, "L", "N")
    assert rfp.pftrf(r) == 0
    assert _backward_error(P, r.data, a, n, "L", "N") <= 10
    b = torch.randn(nrhs, n, dtype=torch.float64, device="cuda", generator=g).t()
    x = b.clone()
    rfp.pftrs(r, x)
    res = float((a @ x - b).norm() / (a.norm() * x.norm() * n * 2.0 ** -53))
    assert res <= 10


@pytest.mark.parametrize("n", [1500, 3001])
def test_config5_complex_inverse_columns(P, n):
    """Config 5 shape at reduced n: complex Hermitian, TRANSR='C', UPLO='L',
    A = B B^H / n + I, pftrf -> pftri, ||A Y - I[:, J]|| on 256 columns."""
    conv, rfp = P.convert, P.rfp
    g = torch.Generator(device="cuda").manual_seed(n)
    s = 0.5 ** 0.5
    bm = torch.complex(torch.randn(n, n, dtype=torch.float64, device="cuda", generator=g) * s,
                       torch.randn(n, n, dtype=torch.float64, device="cuda", generator=g) * s)
    a = bm @ bm.mH / n
    a.diagonal().add_(1.0)
    r = conv.trttf(a, "L", "C")
    assert rfp.pftrf(r) == 0
    assert rfp.pftri(r) == 0
    full = conv.tfttr(r)
    inv = torch.tril(full) + torch.tril(full, -1).mH
    J = torch.randperm(n, generator=torch.Generator().manual_seed(1))[:256].cuda()
    E = a @ inv[:, J]
    E[J, torch.arange(256, device="cuda")] -= 1.0
    assert float(E.abs().max()) <= 1e-12


# ---------------------------------------------------------------- SURVEY 8(f) rows
from tests.conftest import next_row_cases  # noqa: E402

with np.load(GOLDEN) as _z2:
    NEXT = next_row_cases({k: None for k in _z2.files})


@pytest.mark.parametrize("key,dt,uplo,transr,n", NEXT, ids=[c[0] for c in NEXT])
def test_next_rows_match_reference(P, golden, key, dt, uplo, transr, n):
    conv, rfp, layout = P.convert, P.rfp, P.layout
    cplx = dt == "c128"
    d = layout.make_descriptor(n, uplo, transr)
    f = conv.RfpTriangle(golden[f"tfsm_{key}_factor"], d)
    for side in "LR":
        for trans in "NTC":
            for diag in "NU":
                b = torch.from_numpy(golden[f"tfsm_{key}_{side}{trans}{diag}_B"]).cuda()
                alpha = (1.5 - 0.5j) if cplx else 1.5
                rfp.tfsm(transr, side, uplo, trans, diag, b.shape[0], b.shape[1], alpha, f, b)
                assert rel(b, golden[f"tfsm_{key}_{side}{trans}{diag}_X"]) <= TOL, (side, trans, diag)
    for trans in "NC":
        c = conv.RfpTriangle(golden[f"sfrk_{key}_{trans}_C0"], d)
        rfp.sfrk_hfrk(transr, uplo, trans, n, 5, -0.75, golden[f"sfrk_{key}_{trans}_A"], 1.25, c)
        assert rel(c.data, golden[f"sfrk_{key}_{trans}_C"]) <= TOL
    r = conv.RfpTriangle(golden[f"lansf_{key}_rfp"], d)
    got = [rfp.lansf(nm, r) for nm in "M1IF"]
    assert np.allclose(got, golden[f"lansf_{key}"], rtol=1e-12, atol=0)


def test_next_rows_large_vs_oracle(P):
    """Recursive sizes for tfsm / sfrk_hfrk / lansf against the oracle, plus
    the singular-index re-basing of tfsm (rfp.py:46-52)."""
    conv, rfp, kernels = P.convert, P.rfp, P.kernels
    for n, uplo, transr, cplx in [(700, "L", "N", False), (513, "U", "T", True), (1100, "U", "N", False)]:
        a = O.spd_matrix(n, n, "n", complex_=cplx)
        buf = O.trttf(a, uplo, transr)
        f = buf.copy()
        assert O.pftrf(f, n, uplo, transr) == 0
        fr = conv.RfpTriangle(f, P.layout.make_descriptor(n, uplo, transr))
        g = np.random.default_rng(n)
        for side, trans in [("L", "N"), ("R", "C"), ("L", "T"), ("R", "N")]:
            shape = (n, 9) if side == "L" else (9, n)
            b = np.asfortranarray(g.standard_normal(shape) + (1j * g.standard_normal(shape) if cplx else 0))
            xo = b.copy(order="F")
            O.tfsm(f, n, uplo, transr, side, trans, "N", 0.5, xo)
            x = torch.from_numpy(b).cuda()
            rfp.tfsm(transr, side, uplo, trans, "N", shape[0], shape[1], 0.5, fr, x)
            assert rel(x, xo) <= TOL
        k = 37
        ga = np.asfortranarray(g.standard_normal((n, k)) + (1j * g.standard_normal((n, k)) if cplx else 0))
        co = buf.copy()
        O.sfrk_hfrk(co, n, uplo, transr, "N", k, 2.0, ga, -0.5, cplx)
        c = conv.RfpTriangle(buf.copy(), P.layout.make_descriptor(n, uplo, transr))
        rfp.sfrk_hfrk(transr, uplo, "N", n, k, 2.0, ga, -0.5, c)
        assert rel(c.data, co) <= TOL
        for nm in "M1IF":
            assert rfp.lansf(nm, c) == pytest.approx(O.lansf(nm, co, n, uplo, transr), rel=1e-12)
    # singular triangle: global index of the zero diagonal (T2 block, L layout)
    n = 150
    a = O.spd_matrix(n, 3, "n")
    f = O.trttf(a, "L", "N")
    assert O.pftrf(f, n, "L", "N") == 0
    ds = O.desc(n, "L", "N")
    t1, t2, s1 = O.blocks(f, ds)
    t2[10, 10] = 0.0
    fr = conv.RfpTriangle(f, P.layout.make_descriptor(n, "L", "N"))
    b = torch.ones(n, 2, dtype=torch.float64, device="cuda")
    with pytest.raises(kernels.SingularMatrixError) as e:
        rfp.tfsm("N", "L", "L", "N", "N", n, 2, 1.0, fr, b)
    with pytest.raises(O.OracleSingular) as eo:
        O.tfsm(f, n, "L", "N", "L", "N", "N", 1.0, np.ones((n, 2), order="F"))
    assert e.value.index == eo.value.index == ds.n1 + 11


# ---------------------------------------------------------------- SURVEY 8(f) row 4
def test_packed_cholesky_vs_reference(P, golden):
    """pptrf_ref / pptrs_ref (packed.py:70-146) through the C ABI against the
    reference's own outputs: factors and solutions within 1e-10, failure
    index identical; host RHS solved in place."""
    conv, packed = P.convert, P.packed
    keys = sorted(k[:-5] for k in golden if k.startswith("pp_") and k.endswith("_info"))
    assert len(keys) >= 30
    for key in keys:
        _, dt, uplo, nn, *rest = key.split("_")
        n = int(nn[1:])
        p = conv.PackedTriangle(golden[key + "_P"].copy(), n, uplo)
        assert packed.pptrf_ref(p) == int(golden[key + "_info"]), key
        if rest:
            continue
        assert rel(p.data, golden[key + "_F"]) <= TOL, key
        x = golden[key + "_B"].copy(order="F")
        packed.pptrs_ref(p, x)  # host array, written back
        assert rel(x, golden[key + "_X"]) <= TOL, key
        xd = torch.from_numpy(golden[key + "_B"].copy()).cuda()
        packed.pptrs_ref(p, xd[:, 0])  # 1-D device RHS
        assert rel(xd[:, 0], golden[key + "_X"][:, 0]) <= TOL, key
    with pytest.raises(ValueError):
        packed.pptrs_ref(conv.PackedTriangle(golden[keys[-1] + "_P"], int(keys[-1].split("_")[3][1:]),
                                             keys[-1].split("_")[2]), torch.ones(3, 2, device="cuda"))


@pytest.mark.parametrize("uplo", "LU")
@pytest.mark.parametrize("cplx", [False, True])
def test_packed_cholesky_large_vs_oracle(P, uplo, cplx):
    conv, packed = P.convert, P.packed
    n = 700
    a = O.spd_matrix(n, 11, "n", complex_=cplx)
    po = O.pack(a, uplo)
    pg = conv.PackedTriangle(po.copy(), n, uplo)
    assert O.pptrf(po, n, uplo) == 0 == packed.pptrf_ref(pg)
    assert rel(pg.data, po) <= TOL
    b = np.asfortranarray(np.random.default_rng(2).standard_normal((n, 5)) + (1j if cplx else 0))
    xo = b.copy(order="F")
    O.pptrs(po, n, uplo, xo)
    xg = torch.from_numpy(b.copy()).cuda()
    packed.pptrs_ref(pg, xg)
    assert rel(xg, xo) <= TOL


@pytest.mark.parametrize("uplo", "LU")
@pytest.mark.parametrize("transr", "NT")
@pytest.mark.parametrize("n", [7, 130, 601, 1100, 2049])
def test_pftrf_from_host_streamed(P, uplo, transr, n):
    """The streamed host->device pftrf gives the device pftrf's factor and
    failure index: bit-identical for complex data; for real data with the
    leading block <= 4096 the device path factors [T1; S1] (or [T1; S1^T] for
    'U') as one panel while the streamed one keeps the separate S1 solve
    (same math, other summation order), so within TOL."""
    conv, rfp = P.convert, P.rfp
    for cplx in (False, True):
        a = O.spd_matrix(n, 3 + n, "n", complex_=cplx)
        buf = O.trttf(a, uplo, transr)
        host = torch.from_numpy(buf.copy()).pin_memory()
        r, info = rfp.pftrf_from_host(host, n, uplo, transr)
        ref = conv.RfpTriangle(buf.copy(), P.layout.make_descriptor(n, uplo, transr))
        assert info == 0 == rfp.pftrf(ref)
        if cplx:
            assert bits(r.data) == bits(ref.data)
        else:
            assert rel(r.data, ref.data.cpu().numpy()) <= TOL
        assert r.state is conv.FactorState.CHOLESKY
    bad = O.trttf(np.eye(n) - 2.0 * (np.arange(n) == n // 2)[:, None] * np.eye(n), uplo, transr)
    _, info = rfp.pftrf_from_host(bad, n, uplo, transr)
    assert info == n // 2 + 1


def test_phase_clock_times_srpa_steps(P):
    """rfpk_phase_clock / rfpk_phase_time: event pairs around the SRPA steps of
    direct calls, read without synchronising the calls themselves."""
    import ctypes
    from paper_0901_1696_b200 import _capi
    lib = _capi.lib()
    n = 1037  # an order no other test uses: the first call is direct (not a graph replay)
    a = O.spd_matrix(n, 9, "n")
    lib.rfpk_phase_clock(1)
    r = P.convert.trttf(a, "L", "N")
    assert P.rfp.pftrf(r) == 0  # first call of this shape: direct (the one-launch chain)
    tot, cnt = ctypes.c_double(0), ctypes.c_int64(0)
    assert lib.rfpk_phase_time(b"pftrf potrf(T1)+trsm(S1)+syrk(T2)+potrf(T2)", ctypes.byref(tot),
                               ctypes.byref(cnt)) == 0
    assert cnt.value >= 1 and tot.value > 0
    assert lib.rfpk_phase_time(b"kernel tile_potrf 1037x1037", ctypes.byref(tot),
                               ctypes.byref(cnt)) == 0
    assert cnt.value >= 1 and tot.value > 0
    with _capi.tuning(panel_max=0):  # the step-by-step SRPA sequence
        r = P.convert.trttf(a, "L", "N")
        assert P.rfp.pftrf(r) == 0
    assert lib.rfpk_phase_time(b"pftrf syrk(T2)", ctypes.byref(tot), ctypes.byref(cnt)) == 0
    assert cnt.value >= 1 and tot.value > 0
    assert lib.rfpk_phase_time(b"no such phase", ctypes.byref(tot), ctypes.byref(cnt)) == 1
    lib.rfpk_phase_clock(0)


def test_concurrent_host_threads_on_own_streams(P):
    """Four host threads, each on its own CUDA stream, factor and solve
    different matrices at the same time (tile kernels with per-call sync
    buffers, thread-local graph capture, per-thread info buffers)."""
    import threading
    conv, rfp = P.convert, P.rfp
    errs, res = [], {}

    def work(tid):
        try:
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                for rep in range(3):
                    n = 700 + 37 * tid
                    uplo, transr = "LU"[tid % 2], "NT"[(tid // 2) % 2]
                    a = O.spd_matrix(n, 100 + tid, "n")
                    r = conv.trttf(a, uplo, transr)
                    assert rfp.pftrf(r) == 0
                    b = np.random.default_rng(tid).standard_normal((n, 3))
                    x = torch.from_numpy(b.copy()).cuda()
                    rfp.pftrs(r, x)
                    s.synchronize()
                    res[(tid, rep)] = float(np.abs(a @ x.cpu().numpy() - b).max() / np.abs(b).max())
        except Exception as e:  # pragma: no cover - surfaced below
            errs.append(repr(e))

    th = [threading.Thread(target=work, args=(t,)) for t in range(4)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs, errs
    assert len(res) == 12 and max(res.values()) < 1e-9


# ---------------------------------------------------------------- SPEC acceptance checks
@pytest.mark.slow
def test_reentrant_large_orders_on_own_streams(P):
    """Re-entrancy at orders where the library forks its own side streams:
    n1 > 4096, so pftrf runs potrf(T1) || S1 solve as two spin-coupled
    launches and pfsv runs pftrs part 1 beside potrf(T2).  Four host threads,
    each on its own stream, run pftrf and pfsv on their own matrices five
    times; every result must be bit-identical to the same call made alone
    (single thread, nothing else on the device)."""
    import threading
    conv, rfp = P.convert, P.rfp
    cases = [(8194, "L", "N"), (9001, "L", "N"), (9500, "U", "N"), (10000, "L", "T")]
    inputs_ = []
    for k, (n, uplo, transr) in enumerate(cases):
        g = torch.Generator(device="cuda").manual_seed(50 + k)
        bm = torch.randn(n, n, dtype=torch.float64, device="cuda", generator=g)
        a = bm @ bm.t() / n
        a.diagonal().add_(1.0)
        del bm
        src = conv.trttf(a, uplo, transr).data
        b = torch.randn(64, n, dtype=torch.float64, device="cuda", generator=g).t()
        inputs_.append((src, b))
        del a

    def run(k):
        n, uplo, transr = cases[k]
        src, b = inputs_[k]
        d = P.layout.make_descriptor(n, uplo, transr)
        r1 = conv.RfpTriangle(src.clone(), d)
        assert rfp.pftrf(r1) == 0
        r2 = conv.RfpTriangle(src.clone(), d)
        x = b.clone()
        assert rfp.pfsv(r2, x) == 0
        torch.cuda.current_stream().synchronize()
        return r1.data, r2.data, x

    alone = [run(k) for k in range(len(cases))]
    torch.cuda.synchronize()
    errs = []

    def work(k):
        try:
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                for rep in range(5):
                    got = run(k)
                    for u, v in zip(got, alone[k]):
                        if not torch.equal(u, v):
                            errs.append(f"thread {k} rep {rep}: result differs")
        except Exception as e:  # pragma: no cover - surfaced below
            errs.append(repr(e))

    th = [threading.Thread(target=work, args=(k,)) for k in range(len(cases))]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    assert not any(t.is_alive() for t in th), "a thread hung"
    assert not errs, errs


def test_stream_of_another_device_is_served_on_its_device(P):
    """The C ABI switches to the device owning the caller's stream (and back):
    a pftrf on cuda:0's stream issued while another device is current.  With
    one GPU the check is that the current device is restored and the call
    succeeds from a non-default current stream."""
    conv, rfp = P.convert, P.rfp
    n = 300
    a = O.spd_matrix(n, 3, "n")
    f = O.trttf(a, "L", "N")
    assert O.pftrf(f, n, "L", "N") == 0
    ndev = torch.cuda.device_count()
    other = 1 if ndev > 1 else 0
    r = conv.trttf(a, "L", "N")
    s = torch.cuda.Stream(device=0)
    with torch.cuda.device(other):
        with torch.cuda.stream(s):
            assert rfp.pftrf(r) == 0
        assert torch.cuda.current_device() == other
    assert rel(r.data, f) <= TOL


@pytest.mark.parametrize("uplo", "LU")
@pytest.mark.parametrize("transr", "NT")
@pytest.mark.parametrize("cplx", [False, True])
def test_poisoned_other_triangle_never_read(P, uplo, transr, cplx):
    """the unused triangle of the full input may hold NaN; trttf
    (and trttp) read only the declared triangle, so the RFP buffer is NaN-free
    and equal to the clean conversion bit for bit."""
    conv, packed = P.convert, P.packed
    n = 67
    a = O.spd_matrix(n, 4, "n", complex_=cplx)
    bad = a.copy()
    iu = np.triu_indices(n, 1) if uplo == "L" else np.tril_indices(n, -1)
    bad[iu] = np.nan
    r = conv.trttf(bad, uplo, transr)
    assert not torch.isnan(r.data).any()
    assert bits(r.data) == bits(conv.trttf(a, uplo, transr).data)
    p = packed.pack(bad, uplo)
    assert not torch.isnan(p.data).any()


@pytest.mark.parametrize("n", [129, 700])
def test_inverse_residual_and_determinism(P, n):
    """||A inv(A) - I||_F <= 1000 n eps, and SPEC.md:440: the same
    input gives bit-identical factor and inverse on repeated runs."""
    conv, rfp, layout = P.convert, P.rfp, P.layout
    eps = 2.0 ** -53
    for uplo, transr in [("L", "N"), ("U", "T")]:
        a = O.spd_matrix(n, 21, "n")
        outs = []
        for rep in range(2):
            r = conv.trttf(a, uplo, transr)
            assert rfp.pftrf(r) == 0
            f = bits(r.data)
            assert rfp.pftri(r) == 0
            outs.append((f, bits(r.data)))
            inv = O.expand_hermitian(r.data.cpu().numpy(), n, uplo, transr)
            res = np.linalg.norm(a @ inv - np.eye(n)) / (n * eps)
            assert res <= 1000, (uplo, transr, res)
        assert outs[0] == outs[1]


@pytest.mark.timeout(300)
@pytest.mark.parametrize("uplo", "LU")
@pytest.mark.parametrize("n", [1100, 2049])
def test_pfsv_from_host_failure_returns(P, uplo, n):
    """A non-PD host problem: the solves skip on info, and the head block's
    per-row-block copies (which wait on the last solve's row counters) must
    still be released -- the call returns the reference's failure index
    (the solution is unspecified on failure, as documented)."""
    conv, rfp = P.convert, P.rfp
    a = O.spd_matrix(n, 17 + n, "n")
    bad = n // 3
    a[bad, bad] = -1.0
    buf = O.trttf(a, uplo, "N")
    want = O.pftrf(buf.copy(), n, uplo, "N")
    assert want == bad + 1
    b = np.random.default_rng(n).standard_normal((n, 7))
    hb = torch.from_numpy(b.T.copy()).pin_memory().t()
    out = torch.from_numpy(np.full((7, n), np.nan)).pin_memory().t()
    r, info = rfp.pfsv_from_host(torch.from_numpy(buf.copy()).pin_memory(), hb, n, uplo, "N",
                                 out=out)
    assert info == want


@pytest.mark.parametrize("uplo", "LU")
@pytest.mark.parametrize("transr", "NT")
@pytest.mark.parametrize("n", [1, 2, 130, 601, 1100, 2049])
def test_pfsv_from_host_overlapped(P, uplo, transr, n):
    """pftrf + pftrs of a host problem with the transfers overlapped: the
    device path's factor (bit-identical for 'U'; within TOL for 'L', where the
    device path may factor [T1; S1] as one panel) and solution."""
    conv, rfp = P.convert, P.rfp
    for cplx in (False, True):
        a = O.spd_matrix(n, 5 + n, "n", complex_=cplx)
        buf = O.trttf(a, uplo, transr)
        g = np.random.default_rng(n)
        b = g.standard_normal((n, 5)) + (1j * g.standard_normal((n, 5)) if cplx else 0)
        hb = torch.from_numpy(b.T.copy()).pin_memory().t()  # pinned, column-major n x 5
        out = torch.from_numpy(np.zeros((5, n), dtype=b.dtype)).pin_memory().t()
        r, info = rfp.pfsv_from_host(torch.from_numpy(buf.copy()).pin_memory(), hb, n, uplo,
                                     transr, out=out)
        assert info == 0
        ref = conv.RfpTriangle(buf.copy(), P.layout.make_descriptor(n, uplo, transr))
        assert rfp.pftrf(ref) == 0
        if cplx:
            assert bits(r.data) == bits(ref.data)
        else:
            assert rel(r.data, ref.data.cpu().numpy()) <= TOL
        xd = torch.from_numpy(b.copy()).cuda()
        rfp.pftrs(ref, xd)
        assert rel(out, xd.cpu()) <= 1e-12
        # numpy in, solved in place; 1-D right-hand side
        bn = np.array(b[:, 0])
        rfp.pfsv_from_host(buf.copy(), bn, n, uplo, transr)
        assert rel(bn, xd[:, 0].cpu()) <= 1e-12


@pytest.mark.parametrize("nrhs", [0, 3, 8])
def test_batched_from_host_pipelined(P, nrhs):
    """The chunked host pipeline gives bit-for-bit the device-resident fused
    kernel's factors, solutions and info (ragged last chunk; nrhs 0 = a 2-D
    (batch, n) right-hand side)."""
    rfp = P.rfp
    n, batch = 64, 37
    bufs = [O.trttf(O.spd_matrix(n, 500 + k, "n"), "U", "N") for k in range(batch)]
    host_arf = torch.from_numpy(np.stack(bufs)).pin_memory()
    g = np.random.default_rng(9)
    if nrhs:
        base = torch.from_numpy(g.standard_normal((batch, nrhs, n))).pin_memory()
        host_b = base.transpose(1, 2)                      # (batch, n, nrhs), unit stride along n
        out = torch.empty_like(base).pin_memory().transpose(1, 2)
    else:
        host_b = torch.from_numpy(g.standard_normal((batch, n))).pin_memory()
        out = torch.empty_like(host_b).pin_memory()
    d_arf, info = rfp.pftrf_pftrs_batched_from_host(host_arf, "N", "U", n, host_b, out=out, chunk=10)
    torch.cuda.synchronize()
    ref_arf = host_arf.cuda()
    ref_b = host_b.cuda()
    ref_info = rfp.pftrf_pftrs_batched(ref_arf, "N", "U", n, ref_b)
    assert torch.equal(info, ref_info) and int(info.abs().sum()) == 0
    assert torch.equal(d_arf, ref_arf)
    assert torch.equal(out, ref_b.cpu())


@pytest.mark.parametrize("transr", "NT")
@pytest.mark.parametrize("bad", [None, 100, 460, 700])
def test_pftrf_panel_path(P, transr, bad):
    """n = 1000 'L': the whole SRPA chain runs as one dataflow launch whose
    region-0 tiles end with a ragged 52-column tile (448..499) before T2's
    tiles restart at 500; factor parity with the oracle, and the reference's
    failure index for a non-PD pivot in T1's full tiles (100), in the ragged
    tile (460) and in T2 (700)."""
    conv, rfp = P.convert, P.rfp
    n = 1000
    a = O.spd_matrix(n, 21, "n")
    if bad is not None:
        a[:, bad] = 0.0
        a[bad, :] = 0.0
        a[bad, bad] = -1.0
    buf = O.trttf(a, "L", transr)
    f = buf.copy()
    want = O.pftrf(f, n, "L", transr)
    r = conv.trttf(a, "L", transr)
    assert rfp.pftrf(r) == want
    if bad is None:
        assert want == 0
        assert rel(r.data, f) <= TOL
    else:
        assert want == bad + 1


def _kernel_launches(prefix, fn):
    """Launches of library kernels whose kernel-clock label starts with
    ``prefix`` (e.g. "kernel tile_copy") during fn(), and fn()'s result."""
    from paper_0901_1696_b200 import _capi
    torch.cuda.synchronize()
    with _capi.phase_clock() as pc:
        out = fn()
        torch.cuda.synchronize()
    return out, sum(c for lab, (_, c) in pc.table().items() if lab.startswith(prefix))


def _phase_count(label, fn):
    """Number of SRPA phases named ``label`` the phase clock saw during fn()
    (direct calls only -- the forced paths below are never graph-captured
    because every call gets fresh buffers)."""
    import ctypes
    from paper_0901_1696_b200 import _capi
    lib = _capi.lib()
    lib.rfpk_phase_clock(1)
    try:
        out = fn()
        ms, cnt = ctypes.c_double(0.0), ctypes.c_int64(0)
        lib.rfpk_phase_time(label.encode(), ctypes.byref(ms), ctypes.byref(cnt))
    finally:
        lib.rfpk_phase_clock(0)
    return out, int(cnt.value)


@pytest.mark.parametrize("uplo", "LU")
@pytest.mark.parametrize("transr", "NT")
@pytest.mark.parametrize("n", [777, 1299])
@pytest.mark.parametrize("cplx", [False, True])
def test_potrf_row_major_block_copy(P, uplo, transr, n, cplx):
    """A diagonal block whose lower view is row-major (T2 for TRANSR='N', T1
    for 'T') is factored in a column-major copy (forced here with tuning
    t2_copy_min=64 -- the copies show up as extra launches; default from
    order 2048 up, real data only -- the complex cases check that the direct
    path is unaffected): factor within TOL of the oracle, and failure indices
    inside either block are the reference's."""
    from paper_0901_1696_b200 import _capi
    conv, rfp = P.convert, P.rfp
    a = O.spd_matrix(n, 31 + n, "n", complex_=cplx)
    f = O.trttf(a, uplo, transr)
    assert O.pftrf(f, n, uplo, transr) == 0
    with _capi.tuning(panel_max=0):  # the step-by-step sequence (potrf_block)
        info0, plain = _kernel_launches("kernel tile_copy",
                                        lambda: rfp.pftrf(conv.trttf(a, uplo, transr)))
    with _capi.tuning(t2_copy_min=64, panel_max=0):
        r = conv.trttf(a, uplo, transr)
        info, forced = _kernel_launches("kernel tile_copy", lambda: rfp.pftrf(r))
        assert info == info0 == 0
        assert rel(r.data, f) <= TOL
        # real data: the row-major block (T2's lower view for TRANSR='N', T1's
        # for 'T', outside the one-launch paths) goes through the copy (two
        # more tile copies); complex never does
        assert forced - plain == (0 if cplx else 2)
        for k in (2, n - 3):  # inside the leading block, inside the trailing one
            bad = a.copy()
            bad[k, k] = -1.0
            fb = O.trttf(bad, uplo, transr)
            want = O.pftrf(fb, n, uplo, transr)
            assert want == k + 1
            rb = conv.trttf(bad, uplo, transr)
            assert rfp.pftrf(rb) == want


@pytest.mark.parametrize("uplo", "LU")
def test_potrf_trsm_overlap_info_and_factor(P, uplo):
    """Above the panel limit (forced low: tuning panel_max=256) potrf(T1) and
    the S1 solve run as two concurrent launches, the solve gated on the
    potrf's diagonal flags (the phase clock sees the overlapped phase; 'U'
    keeps the sequence, its column-major-B solve does not fit beside the
    potrf): factor within TOL of the oracle, and a failure inside T1 (every
    gated solve task must then exit) returns the reference's index without
    hanging."""
    from paper_0901_1696_b200 import _capi
    conv, rfp = P.convert, P.rfp
    n = 1403
    a = O.spd_matrix(n, 99, "n")
    f = O.trttf(a, uplo, "N")
    assert O.pftrf(f, n, uplo, "N") == 0
    with _capi.tuning(panel_max=256):
        r = conv.trttf(a, uplo, "N")
        info, seen = _phase_count("pftrf potrf(T1)||trsm(S1)", lambda: rfp.pftrf(r))
        assert info == 0
        assert seen == (1 if uplo == "L" else 0)
        assert rel(r.data, f) <= TOL
        for k in (1, 300, 650):
            bad = a.copy()
            bad[k, k] = -1.0
            want = O.pftrf(O.trttf(bad, uplo, "N"), n, uplo, "N")
            assert want == k + 1
            assert rfp.pftrf(conv.trttf(bad, uplo, "N")) == want


@pytest.mark.parametrize("uplo", "LU")
@pytest.mark.parametrize("transr", "NT")
@pytest.mark.parametrize("n", [1, 130, 1501, 2049])
@pytest.mark.parametrize("cplx", [False, True])
def test_pfsv_device_matches_pftrf_pftrs(P, uplo, transr, n, cplx):
    """rfp.pfsv (the first T1 solve and the S1 product run beside potrf(T2);
    forced from T2 order 64 here, and the phase clock must see that phase
    whenever T2 reaches it) gives pftrf + pftrs's factor and solution within
    TOL of the oracle; a failing factorization leaves b untouched and returns
    the reference's index."""
    from paper_0901_1696_b200 import _capi
    # (panel_max=0: the step-by-step sequence whose potrf(T2) the solve
    # overlaps; the one-launch chain is covered by test_pfsv_fused_chain)
    with _capi.tuning(pfsv_overlap_min=64, panel_max=0):
        _pfsv_case(P, uplo, transr, n, cplx)


@pytest.mark.parametrize("uplo", "LU")
@pytest.mark.parametrize("transr", "NT")
@pytest.mark.parametrize("n", [128, 130, 257, 1501, 2049, 4001])
def test_pfsv_fused_chain(P, uplo, transr, n):
    """Real mid orders factor through the one-launch SRPA chain (every tile of
    T1, S, T2 in one dataflow kernel; the phase clock sees that phase and no
    separate syrk(T2) step); pfsv then solves after it: factor and solution
    within TOL of the oracle, failure index inside T2 the reference's."""
    conv, rfp = P.convert, P.rfp
    a = O.spd_matrix(n, 77 + n, "n")
    f = O.trttf(a, uplo, transr)
    assert O.pftrf(f, n, uplo, transr) == 0
    rng = np.random.default_rng(n + 1)
    bh = rng.standard_normal((n, 5))
    xo = np.asfortranarray(bh.copy())
    O.pftrs(f, n, uplo, transr, xo)
    r = conv.trttf(a, uplo, transr)
    b = torch.from_numpy(np.asfortranarray(bh)).cuda()
    info, seen = _phase_count("pftrf potrf(T1)+trsm(S1)+syrk(T2)+potrf(T2)",
                              lambda: rfp.pfsv(r, b))
    assert info == 0 and seen == 1
    assert rel(r.data, f) <= TOL
    assert rel(b, xo) <= TOL
    bad = a.copy()
    bad[n - 2, n - 2] = -1.0
    want = O.pftrf(O.trttf(bad, uplo, transr), n, uplo, transr)
    assert rfp.pftrf(conv.trttf(bad, uplo, transr)) == want == n - 1


def _pfsv_case(P, uplo, transr, n, cplx):
    conv, rfp = P.convert, P.rfp
    a = O.spd_matrix(n, 5 + n, "n", complex_=cplx)
    f = O.trttf(a, uplo, transr)
    assert O.pftrf(f, n, uplo, transr) == 0
    rng = np.random.default_rng(n)
    bh = rng.standard_normal((n, 9)) + (1j * rng.standard_normal((n, 9)) if cplx else 0)
    xo = np.asfortranarray(bh.copy())
    O.pftrs(f, n, uplo, transr, xo)
    r = conv.trttf(a, uplo, transr)
    b = torch.from_numpy(np.asfortranarray(bh)).cuda()
    info, seen = _phase_count("pftrf potrf(T2)||pftrs(T1,S1)", lambda: rfp.pfsv(r, b))
    assert info == 0
    t2_order = n // 2 if uplo == "L" else (n + 1) // 2
    assert seen == (1 if t2_order >= 64 and n > 1 else 0)
    assert r.state is conv.FactorState.CHOLESKY
    assert rel(r.data, f) <= TOL
    assert rel(b, xo) <= TOL
    if n > 2:
        bad = a.copy()
        bad[n - 2, n - 2] = -1.0
        want = O.pftrf(O.trttf(bad, uplo, transr), n, uplo, transr)
        rb = conv.trttf(bad, uplo, transr)
        b2 = torch.from_numpy(np.asfortranarray(bh)).cuda()
        assert rfp.pfsv(rb, b2) == want > 0
        assert rb.state is conv.FactorState.UNFACTORED
        assert torch.equal(b2.cpu(), torch.from_numpy(np.asfortranarray(bh)))


@pytest.mark.parametrize("uplo,transr,cplx", [("L", "N", False), ("U", "T", True), ("U", "N", False)])
def test_banded_triangular_gemm_orders(P, uplo, transr, cplx):
    """sfrk_hfrk (SYRK/HERK on T1 and T2 + GEMM on S1) at n = 3300, where each
    triangle spans 26 tile rows -- two bands of the banded tile order, the
    second partial -- against the oracle; then pftrf (SYRK of T2 in the same
    order) and pftrs(300) (narrow full GEMMs in their banded order)."""
    conv, rfp = P.convert, P.rfp
    n, k = 3300, 40
    a = O.spd_matrix(n, 17, "n", complex_=cplx)
    buf = O.trttf(a, uplo, transr)
    g = np.random.default_rng(5)
    ga = np.asfortranarray(g.standard_normal((n, k)) + (1j * g.standard_normal((n, k)) if cplx else 0))
    co = buf.copy()
    O.sfrk_hfrk(co, n, uplo, transr, "N", k, 2.0, ga, -0.5, cplx)
    c = conv.RfpTriangle(buf.copy(), P.layout.make_descriptor(n, uplo, transr))
    rfp.sfrk_hfrk(transr, uplo, "N", n, k, 2.0, ga, -0.5, c)
    assert rel(c.data, co) <= TOL
    f = buf.copy()
    assert O.pftrf(f, n, uplo, transr) == 0
    r = conv.trttf(a, uplo, transr)
    assert rfp.pftrf(r) == 0
    assert rel(r.data, f) <= TOL
    bh = g.standard_normal((n, 300)) + (1j * g.standard_normal((n, 300)) if cplx else 0)
    xo = np.asfortranarray(bh.copy())
    O.pftrs(f, n, uplo, transr, xo)
    x = torch.from_numpy(np.asfortranarray(bh)).cuda()
    rfp.pftrs(r, x)
    assert rel(x, xo) <= TOL
