"""Generate golden vectors by running the REFERENCE implementation.

Run in the build container only (it imports /root/reference, which does not
exist on the GPU box):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Writes ``tests/golden/golden.npz``.  The inputs are seeded
(``numpy.random.default_rng``) so the fixtures are reproducible; each entry
holds the reference's own outputs of trttf/tfttr/pack/tpttf/tfttp, pftrf
(+info), pftrs, tftri and pftri for one (dtype, uplo, transr, n) case, and a
set of non-positive-definite cases pinning the reference's failure index.
"""

import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from rfpk import convert, packed, rfp  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def spd(n, seed, cplx):
    rng = np.random.default_rng(seed)
    if cplx:
        s = np.sqrt(0.5)
        b = rng.standard_normal((n, n)) * s + 1j * (rng.standard_normal((n, n)) * s)
    else:
        b = rng.standard_normal((n, n))
    return np.asfortranarray(b @ np.conj(b.T) + n * np.eye(n))


def rhs(n, nrhs, seed, cplx):
    rng = np.random.default_rng(seed + 1000)
    b = rng.standard_normal((n, nrhs))
    if cplx:
        b = b + 1j * rng.standard_normal((n, nrhs))
    return np.asfortranarray(b)


def case(out, n, uplo, transr, cplx, nrhs=3, seed=None):
    seed = 1234 + 7 * n if seed is None else seed
    key = f"{'c128' if cplx else 'f64'}_{uplo}{transr}_n{n}"
    a = spd(n, seed, cplx)
    r = convert.trttf(a, uplo, transr)
    out[key + "_A"] = a
    out[key + "_rfp"] = r.data.copy()
    out[key + "_tfttr"] = convert.tfttr(r)
    p = packed.pack(a, uplo)
    out[key + "_packed"] = p.data.copy()
    out[key + "_tpttf"] = convert.tpttf(p, transr).data.copy()
    out[key + "_tfttp"] = convert.tfttp(r).data.copy()
    f = r.copy()
    out[key + "_pftrf_info"] = np.array(rfp.pftrf(f))
    out[key + "_factor"] = f.data.copy()
    b = rhs(n, nrhs, seed, cplx)
    out[key + "_B"] = b.copy()
    x = b.copy(order="F")
    rfp.pftrs(f, x)
    out[key + "_X"] = x
    ti = f.copy()
    out[key + "_tftri_info"] = np.array(rfp.tftri(ti))
    out[key + "_tftri"] = ti.data.copy()
    inv = f.copy()
    out[key + "_pftri_info"] = np.array(rfp.pftri(inv))
    out[key + "_pftri"] = inv.data.copy()


def next_rows(out, n, uplo, transr, cplx):
    """tfsm (all side/trans/diag), sfrk_hfrk, lansf."""
    key = f"{'c128' if cplx else 'f64'}_{uplo}{transr}_n{n}"
    a = spd(n, 4321 + n, cplx)
    r = convert.trttf(a, uplo, transr)
    f = r.copy()
    assert rfp.pftrf(f) == 0
    rng = np.random.default_rng(77 + n)
    for side in "LR":
        for trans in "NTC":
            for diag in "NU":
                shape = (n, 3) if side == "L" else (3, n)
                b = rng.standard_normal(shape) + (1j * rng.standard_normal(shape) if cplx else 0)
                b = np.asfortranarray(b)
                x = b.copy(order="F")
                alpha = (1.5 - 0.5j) if cplx else 1.5
                rfp.tfsm(transr, side, uplo, trans, diag, x.shape[0], x.shape[1], alpha, f, x)
                out[f"tfsm_{key}_{side}{trans}{diag}_B"] = b
                out[f"tfsm_{key}_{side}{trans}{diag}_X"] = x
    out[f"tfsm_{key}_factor"] = f.data.copy()
    for trans in "NC":
        kk = 5
        g = rng.standard_normal((n, kk) if trans == "N" else (kk, n))
        if cplx:
            g = g + 1j * rng.standard_normal(g.shape)
        c = r.copy()
        rfp.sfrk_hfrk(transr, uplo, trans, n, kk, -0.75, g, 1.25, c)
        out[f"sfrk_{key}_{trans}_A"] = g
        out[f"sfrk_{key}_{trans}_C0"] = r.data.copy()
        out[f"sfrk_{key}_{trans}_C"] = c.data.copy()
    out[f"lansf_{key}"] = np.array([rfp.lansf(nm, r) for nm in "M1IF"])
    out[f"lansf_{key}_rfp"] = r.data.copy()


def packed_chol(out, n, uplo, cplx, fail_k=None):
    """pptrf_ref / pptrs_ref (packed.py:70-146)."""
    key = f"pp_{'c128' if cplx else 'f64'}_{uplo}_n{n}" + (f"_k{fail_k}" if fail_k is not None else "")
    a = spd(n, 555 + n, cplx)
    if fail_k is not None:
        a[fail_k, fail_k] = -1.0
    p = packed.pack(a, uplo)
    out[key + "_P"] = p.data.copy()
    f = p.copy()
    out[key + "_info"] = np.array(packed.pptrf_ref(f))
    out[key + "_F"] = f.data.copy()
    if fail_k is None:
        b = rhs(n, 4, 555 + n, cplx)
        x = b.copy(order="F")
        packed.pptrs_ref(f, x)
        out[key + "_B"] = b
        out[key + "_X"] = x


def failing(out, n, uplo, transr, cplx, k, nan=False):
    """A = I + small symmetric noise with pivot k (0-based) made negative."""
    a = np.eye(n, dtype=np.complex128 if cplx else np.float64)
    rng = np.random.default_rng(99 + n + k)
    noise = 0.01 * rng.standard_normal((n, n))
    a = a + (noise + noise.T) / 2
    a[k, k] = np.nan if nan else -1.0
    a = np.asfortranarray(a)
    key = f"fail_{'c128' if cplx else 'f64'}_{uplo}{transr}_n{n}_k{k}{'_nan' if nan else ''}"
    r = convert.trttf(a, uplo, transr)
    out[key + "_rfp"] = r.data.copy()
    out[key + "_info"] = np.array(rfp.pftrf(r))


def main():
    out = {}
    small = [0, 1, 2, 3, 4, 5, 6, 7, 8, 17, 40, 41]
    for cplx in (False, True):
        for uplo in "LU":
            for transr in "NT":
                for n in small:
                    case(out, n, uplo, transr, cplx)
    for n, uplo, transr, cplx in [(130, "L", "N", False), (129, "U", "T", False),
                                  (130, "U", "N", False), (129, "L", "T", False),
                                  (130, "L", "T", True), (129, "U", "N", True)]:
        case(out, n, uplo, transr, cplx, nrhs=5)
    for cplx in (False, True):
        for uplo in "LU":
            for transr in "NT":
                for n in (1, 6, 7, 40, 41):
                    next_rows(out, n, uplo, transr, cplx)
    for cplx in (False, True):
        for uplo in "LU":
            for transr in "NT":
                for n, k in [(7, 2), (7, 5), (40, 3), (40, 33), (41, 20), (41, 21)]:
                    failing(out, n, uplo, transr, cplx, k)
                failing(out, 40, uplo, transr, cplx, 25, nan=True)
    for cplx in (False, True):
        for uplo in "LU":
            for n in (0, 1, 2, 5, 17, 40, 41, 130):
                packed_chol(out, n, uplo, cplx)
            packed_chol(out, 41, uplo, cplx, fail_k=20)
    # SPEC.md:269-271 / :310 known answers
    two = convert.trttf(np.array([[4.0, 0.0], [2.0, 5.0]]), "L", "N")
    out["spec_n2_rfp"] = two.data.copy()
    rfp.pftrf(two)
    out["spec_n2_factor"] = two.data.copy()
    rfp.pftri(two)
    out["spec_n2_inverse_full"] = convert.tfttr(two)
    bad = convert.trttf(np.array([[1.0, 0.0], [2.0, 1.0]]), "L", "N")
    out["spec_n2_bad_info"] = np.array(rfp.pftrf(bad))
    np.savez_compressed(os.path.join(HERE, "golden.npz"), **out)
    print(f"wrote {len(out)} arrays")


if __name__ == "__main__":
    main()
