"""CPU ORACLE -- TEST INFRASTRUCTURE ONLY.

This module is the parity checker for the B200 RFPF path.  It is a NumPy
restatement of the reference algorithm (``/root/reference/pkg/src/rfpk``):
the SRPA decomposition of pftrf/pftrs/tftri/pftri into full-format kernels
on the T1/T2/S1 blocks, and blocked (nb = 64) full-format kernels whose
inner diagonal blocks are unblocked row/column loops, exactly as the
reference organises its work.  Only ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py`` (its ``cpu_baseline`` leg and ``--impl reference`` arm)
may import it -- never the product package, which has no CPU fallback.

Pinning: ``tests/test_oracle.py`` checks every function here against
golden vectors produced by the reference itself
(``tests/golden/make_golden.py`` imports /root/reference in the build
container) and against the SPEC.md / doctest known answers; conversions are
bit-exact, arithmetic within 1e-12 relative.

Reference citations are given per function as ``file:line``.
"""

from __future__ import annotations

import os
from collections import namedtuple

import numpy as np

NB = max(1, int(os.environ.get("RFPK_NB", "64")))   # kernels.py:32-33
PANEL = 256                                            # kernels.py:35

Desc = namedtuple("Desc", "n n1 n2 nt ldar uplo transr d")


class OracleSingular(Exception):
    """Zero diagonal in a non-unit triangular solve (kernels.py:38-46)."""

    def __init__(self, index):
        super().__init__(f"zero diagonal entry at position {index}")
        self.index = int(index)


# ---------------------------------------------------------------------------
# geometry (layout.py:103-163, convert.py:76-87, 142-153)


def desc(n, uplo, transr):
    """layout.py:103-124; transr 'C' is mapped to the reference's 'T'."""
    n = int(n)
    uplo = str(uplo).upper()[:1]
    transr = {"N": "N", "T": "T", "C": "T"}[str(transr).upper()[:1]]
    n1 = (n + 1) // 2
    return Desc(n, n1, n - n1, n * (n + 1) // 2, n if n % 2 else n + 1,
                uplo, transr, 0 if n % 2 else 1)


def rect_normal(buf, ds):
    """The ldar x n1 rectangle as a strided view of ``buf`` (convert.py:76-87)."""
    if ds.transr == "N":
        return buf.reshape((ds.ldar, ds.n1), order="F")
    return buf.reshape((ds.n1, ds.ldar), order="F").T


def blocks(buf, ds):
    """(t1, t2, s1) views (convert.py:142-153)."""
    r = rect_normal(buf, ds)
    n1, n2, d = ds.n1, ds.n2, ds.d
    if ds.uplo == "L":
        return r[d:d + n1, :n1], r[:n2, 1 - d:1 - d + n2], r[n1 + d:n1 + d + n2, :n1]
    return r[n2 + 1:2 * n2 + 1, :n2], r[n2:n2 + n1, :n1], r[:n2, :n1]


def _cells(ds):
    """For every buffer slot, the 0-based (i, j) of the triangle element it
    holds (inverse of layout.py:127-163), as two int64 arrays of length nt."""
    n = ds.n
    ii, jj = (np.tril_indices(n) if ds.uplo == "L" else np.triu_indices(n))
    n1, n2, d = ds.n1, ds.n2, ds.d
    if ds.uplo == "L":
        lo = jj < n1
        r = np.where(lo, ii + d, jj - n1)
        c = np.where(lo, jj, ii - n1 + 1 - d)
    else:
        hi = jj >= n2
        r = np.where(hi, ii, jj + n2 + 1)
        c = np.where(hi, jj - n2, ii)
    off = c * ds.ldar + r if ds.transr == "N" else r * n1 + c
    perm_i = np.empty(ds.nt, dtype=np.int64)
    perm_j = np.empty(ds.nt, dtype=np.int64)
    perm_i[off] = ii
    perm_j[off] = jj
    return perm_i, perm_j


def _scalar(a):
    """convert.py:37-43: f64/c128 pass through, other dtypes are cast."""
    a = np.asarray(a)
    if a.dtype in (np.float64, np.complex128):
        return a
    return a.astype(np.complex128 if np.iscomplexobj(a) else np.float64)


# ---------------------------------------------------------------------------
# conversions (convert.py:156-275, packed.py:41-67); verbatim copies


def trttf(a, uplo, transr):
    """full (ld >= n) -> flat RFP buffer (convert.py:156-186)."""
    a = _scalar(a)
    n = a.shape[1]
    ds = desc(n, uplo, transr)
    if n == 0:
        return np.empty(0, a.dtype)
    pi, pj = _cells(ds)
    return a[pi, pj].copy()


def tfttr(buf, n, uplo, transr, ld=None):
    """RFP -> zero-filled (ld, n) Fortran array (convert.py:189-217)."""
    ds = desc(n, uplo, transr)
    ld = n if ld is None else int(ld)
    out = np.zeros((ld, n), dtype=buf.dtype, order="F")
    if n:
        pi, pj = _cells(ds)
        out[pi, pj] = buf
    return out


def packed_offsets(n, uplo):
    """Start of each packed column (convert.py:127-135)."""
    j = np.arange(n, dtype=np.int64)
    return j * n - j * (j - 1) // 2 if uplo == "L" else j * (j + 1) // 2


def _packed_ij(n, uplo):
    """(row, col) of every packed slot in storage order."""
    if uplo == "L":
        cols = np.repeat(np.arange(n), np.arange(n, 0, -1))
        starts = packed_offsets(n, "L")
        rows = np.arange(len(cols)) - starts[cols] + cols
    else:
        cols = np.repeat(np.arange(n), np.arange(1, n + 1))
        starts = packed_offsets(n, "U")
        rows = np.arange(len(cols)) - starts[cols]
    return rows.astype(np.int64), cols.astype(np.int64)


def pack(a, uplo):
    """full -> column-packed triangle (packed.py:41-51)."""
    a = _scalar(a)
    n = a.shape[1]
    r, c = _packed_ij(n, str(uplo).upper()[:1])
    return a[r, c].copy()


def unpack(p, n, uplo, ld=None):
    """packed -> zero-filled full (packed.py:54-67)."""
    ld = n if ld is None else int(ld)
    out = np.zeros((ld, n), dtype=p.dtype, order="F")
    r, c = _packed_ij(n, str(uplo).upper()[:1])
    out[r, c] = p
    return out


def tpttf(p, n, uplo, transr):
    """packed -> RFP (convert.py:220-246)."""
    return trttf(unpack(p, n, uplo), uplo, transr)


def tfttp(buf, n, uplo, transr):
    """RFP -> packed (convert.py:249-275)."""
    return pack(tfttr(buf, n, uplo, transr), uplo)


# ---------------------------------------------------------------------------
# full-format kernels (kernels.py)


def pptrf(p, n, uplo):
    """Unblocked packed Cholesky in place (packed.py:70-108): right-looking
    rank-1 updates of the packed trailing columns for 'L', left-looking
    dot-product columns for 'U'.  Returns 0 or the first failing order."""
    herm = np.iscomplexobj(p)
    st = list(packed_offsets(n, uplo)) + [n * (n + 1) // 2]
    if uplo == "L":
        for j in range(n):
            d = p[st[j]].real if herm else p[st[j]]
            if not d > 0:
                return j + 1
            d = np.sqrt(d)
            p[st[j]] = d
            x = p[st[j] + 1:st[j + 1]]
            x /= d
            for c in range(j + 1, n):
                t = c - j - 1
                p[st[c]:st[c + 1]] -= (np.conj(x[t]) if herm else x[t]) * x[t:]
        return 0
    for j in range(n):
        col = p[st[j]:st[j + 1]]  # rows 0..j of column j
        for t in range(j):
            pc = p[st[t]:st[t + 1]]
            col[t] = (col[t] - np.vdot(pc[:t], col[:t])) / pc[t]
        d = col[j].real if herm else col[j]
        if j:
            d = d - (np.vdot(col[:j], col[:j]).real if herm else col[:j] @ col[:j])
        if not d > 0:
            return j + 1
        col[j] = np.sqrt(d)
    return 0


def pptrs(p, n, uplo, b):
    """Forward/backward substitution from a packed factor, in place on b
    (packed.py:111-146)."""
    bv = b.reshape(-1, 1) if b.ndim == 1 else b
    herm = np.iscomplexobj(p)
    st = list(packed_offsets(n, uplo)) + [n * (n + 1) // 2]
    cj = (lambda v: np.conj(v)) if herm else (lambda v: v)
    if uplo == "L":
        for j in range(n):
            col = p[st[j]:st[j + 1]]
            bv[j] /= col[0]
            bv[j + 1:] -= col[1:, None] * bv[j:j + 1]
        for j in range(n - 1, -1, -1):
            col = p[st[j]:st[j + 1]]
            bv[j] -= cj(col[1:]) @ bv[j + 1:]
            bv[j] /= cj(col[0])
        return
    for j in range(n):
        col = p[st[j]:st[j + 1]]
        bv[j] -= cj(col[:j]) @ bv[:j]
        bv[j] /= cj(col[j])
    for j in range(n - 1, -1, -1):
        col = p[st[j]:st[j + 1]]
        bv[j] /= col[j]
        bv[:j] -= col[:j, None] * bv[j:j + 1]


def _opview(a, trans):
    """op(A) as (view, conjugate?) (kernels.py:78-84 semantics)."""
    if trans == "N":
        return a, False
    return a.T, (trans == "C" and np.iscomplexobj(a))


def gemm(transa, transb, alpha, a, b, beta, c):
    """C <- alpha op(A) op(B) + beta C, column panels of 256 (kernels.py:91-145)."""
    m, n = c.shape
    if m == 0 or n == 0:
        return
    if alpha == 0:
        if beta == 0:
            c[...] = 0
        elif beta != 1:
            c *= beta
        return
    av, ca = _opview(a, transa)
    bv, cb = _opview(b, transb)
    for j0 in range(0, n, PANEL):
        j1 = min(n, j0 + PANEL)
        lhs = np.conj(av) if ca else av
        rhs = np.conj(bv[:, j0:j1]) if cb else bv[:, j0:j1]
        prod = lhs @ rhs
        if alpha != 1:
            prod *= alpha
        tgt = c[:, j0:j1]
        if beta == 0:
            tgt[...] = prod
        else:
            if beta != 1:
                tgt *= beta
            tgt += prod


def _solve_tri_rows(t, x, lower, unit, base):
    """Unblocked substitution, row by row (kernels.py:152-174)."""
    k = t.shape[0]
    order = range(k) if lower else range(k - 1, -1, -1)
    for i in order:
        if not unit:
            piv = t[i, i]
            if piv == 0:
                raise OracleSingular(base + i + 1)
            x[i] /= piv
        if lower and i + 1 < k:
            x[i + 1:] -= np.outer(t[i + 1:, i], x[i])
        elif not lower and i > 0:
            x[:i] -= np.outer(t[:i, i], x[i])


def _trsm_left(lower, unit, t, x, nb, base=0):
    """Blocked left solve with the triangle ``t`` (kernels.py:177-195)."""
    n = t.shape[0]
    if lower:
        for j0 in range(0, n, nb):
            j1 = min(n, j0 + nb)
            _solve_tri_rows(t[j0:j1, j0:j1], x[j0:j1], True, unit, base + j0)
            if j1 < n:
                gemm("N", "N", -1.0, t[j1:, j0:j1], x[j0:j1], 1.0, x[j1:])
    else:
        for j1 in range(n, 0, -nb):
            j0 = max(0, j1 - nb)
            _solve_tri_rows(t[j0:j1, j0:j1], x[j0:j1], False, unit, base + j0)
            if j0 > 0:
                gemm("N", "N", -1.0, t[:j0, j0:j1], x[j0:j1], 1.0, x[:j0])


def trsm(side, uplo, trans, diag, alpha, a, b, nb=None):
    """op(A) X = alpha B (L) or X op(A) = alpha B (R), in place on b
    (kernels.py:198-238)."""
    nb = NB if nb is None else nb
    if b.size == 0:
        return
    if side == "R":
        # X op(A) = B  <=>  op(A)^T X^T = B^T
        if trans == "C" and np.iscomplexobj(a):
            return trsm("L", "U" if uplo == "L" else "L", "C", diag, alpha, a.T, b.T, nb)
        return trsm("L", uplo, "T" if trans == "N" else "N", diag, alpha, a, b.T, nb)
    t, conj = _opview(a, trans)
    lower = (uplo == "L") == (trans == "N")
    if alpha == 0:
        b[...] = 0
        return
    if conj:
        np.conjugate(b, out=b)
        alpha = np.conj(alpha)
    if alpha != 1:
        b *= alpha
    _trsm_left(lower, diag == "U", t, b, nb)
    if conj:
        np.conjugate(b, out=b)


def _trmm_rows(t, x, lower, unit, alpha):
    """Unblocked triangular multiply row by row (kernels.py:245-264)."""
    k = t.shape[0]
    order = range(k - 1, -1, -1) if lower else range(k)
    for i in order:
        acc = (1.0 if unit else t[i, i]) * x[i]
        if lower and i > 0:
            acc = acc + t[i, :i] @ x[:i]
        elif not lower and i + 1 < k:
            acc = acc + t[i, i + 1:] @ x[i + 1:]
        x[i] = acc * alpha if alpha != 1 else acc


def trmm(side, uplo, trans, diag, alpha, a, b, nb=None):
    """B <- alpha op(A) B (L) or alpha B op(A) (R) (kernels.py:267-321)."""
    nb = NB if nb is None else nb
    if b.size == 0:
        return
    if alpha == 0:
        b[...] = 0
        return
    if side == "R":
        if trans == "C" and np.iscomplexobj(a):
            return trmm("L", "U" if uplo == "L" else "L", "C", diag, alpha, a.T, b.T, nb)
        return trmm("L", uplo, "T" if trans == "N" else "N", diag, alpha, a, b.T, nb)
    t, conj = _opview(a, trans)
    lower = (uplo == "L") == (trans == "N")
    unit = diag == "U"
    if conj:
        np.conjugate(b, out=b)
        alpha = np.conj(alpha)
    n = t.shape[0]
    if lower:
        for j1 in range(n, 0, -nb):
            j0 = max(0, j1 - nb)
            _trmm_rows(t[j0:j1, j0:j1], b[j0:j1], True, unit, alpha)
            if j0 > 0:
                gemm("N", "N", alpha, t[j0:j1, :j0], b[:j0], 1.0, b[j0:j1])
    else:
        for j0 in range(0, n, nb):
            j1 = min(n, j0 + nb)
            _trmm_rows(t[j0:j1, j0:j1], b[j0:j1], False, unit, alpha)
            if j1 < n:
                gemm("N", "N", alpha, t[j0:j1, j1:], b[j1:], 1.0, b[j0:j1])
    if conj:
        np.conjugate(b, out=b)


def syrk_herk(uplo, trans, alpha, a, beta, c, herm=False):
    """Declared triangle of C <- alpha G G^(T|H) + beta C, G = A ('N') or
    G = A^(T|H) ('T'/'C'); Hermitian diagonal forced real; the other
    triangle is never touched (kernels.py:328-423)."""
    n = c.shape[0]
    if n == 0:
        return
    g = a if trans == "N" else (np.conj(a.T) if herm else a.T)
    k = g.shape[1]
    lower = uplo == "L"
    if alpha == 0 or k == 0:
        if beta != 1:
            for j in range(n):
                col = c[j:, j] if lower else c[:j + 1, j]
                col[...] = 0 if beta == 0 else col * beta
        return
    gh = np.conj(g.T) if herm else g.T
    for j0 in range(0, n, PANEL):
        j1 = min(n, j0 + PANEL)
        r0, r1 = (j0, n) if lower else (0, j1)
        p = g[r0:r1] @ gh[:, j0:j1]
        w = j1 - j0
        blk = c[j0:j1, j0:j1]
        pd = p[j0 - r0:j0 - r0 + w]
        idx = np.tril_indices(w) if lower else np.triu_indices(w)
        blk[idx] = alpha * pd[idx] + (beta * blk[idx] if beta != 0 else 0)
        if herm and np.iscomplexobj(blk):
            dd = np.arange(w)
            blk[dd, dd] = blk[dd, dd].real
        if lower and j1 < n:
            tgt, src = c[j1:, j0:j1], p[w:]
        elif not lower and j0 > 0:
            tgt, src = c[:j0, j0:j1], p[:j0]
        else:
            continue
        if beta == 0:
            tgt[...] = alpha * src
        else:
            if beta != 1:
                tgt *= beta
            tgt += alpha * src


def _potf2(a, lower, herm, base):
    """Unblocked left-looking Cholesky of a diagonal block; returns 0 or the
    1-based global failing pivot; ``not d > 0`` catches NaN (kernels.py:430-465)."""
    k = a.shape[0]
    for i in range(k):
        v = a[i, :i] if lower else a[:i, i]
        s = np.vdot(v, v).real if herm else v @ v
        d = (a[i, i].real if herm else a[i, i]) - s
        if not d > 0:
            return base + i + 1
        d = np.sqrt(d)
        a[i, i] = d
        if i + 1 < k:
            vc = np.conj(v) if herm else v
            if lower:
                col = a[i + 1:, i]
                if i:
                    col -= a[i + 1:, :i] @ vc
                col /= d
            else:
                row = a[i, i + 1:]
                if i:
                    row -= vc @ a[:i, i + 1:]
                row /= d
    return 0


def potrf(uplo, a, nb=None):
    """Blocked right-looking Cholesky (kernels.py:468-496): L L^H or U^H U."""
    nb = NB if nb is None else nb
    n = a.shape[0]
    herm = np.iscomplexobj(a)
    lower = uplo == "L"
    for j0 in range(0, n, nb):
        j1 = min(n, j0 + nb)
        dblk = a[j0:j1, j0:j1]
        info = _potf2(dblk, lower, herm, j0)
        if info:
            return info
        if j1 < n:
            if lower:
                pan = a[j1:, j0:j1]
                trsm("R", "L", "C", "N", 1.0, dblk, pan, nb)
                syrk_herk("L", "N", -1.0, pan, 1.0, a[j1:, j1:], herm)
            else:
                pan = a[j0:j1, j1:]
                trsm("L", "U", "C", "N", 1.0, dblk, pan, nb)
                syrk_herk("U", "C", -1.0, pan, 1.0, a[j1:, j1:], herm)
    return 0


def _trti2(a, lower, unit, nb):
    """Diagonal-block inverse by solving against I (kernels.py:503-512)."""
    k = a.shape[0]
    e = np.eye(k, dtype=a.dtype)
    _trsm_left(lower, unit, a, e, nb)
    off = 1 if unit else 0
    idx = np.tril_indices(k, -off) if lower else np.triu_indices(k, off)
    a[idx] = e[idx]


def trtri(uplo, diag, a, nb=None):
    """Blocked in-place triangular inverse (kernels.py:515-547)."""
    nb = NB if nb is None else nb
    n = a.shape[0]
    unit = diag == "U"
    if not unit:
        for i in range(n):
            if a[i, i] == 0:
                return i + 1
    if uplo == "U":
        for j0 in range(0, n, nb):
            j1 = min(n, j0 + nb)
            if j0:
                trmm("L", "U", "N", diag, 1.0, a[:j0, :j0], a[:j0, j0:j1], nb)
                trsm("R", "U", "N", diag, -1.0, a[j0:j1, j0:j1], a[:j0, j0:j1], nb)
            _trti2(a[j0:j1, j0:j1], False, unit, nb)
    else:
        for j1 in range(n, 0, -nb):
            j0 = max(0, j1 - nb)
            if j1 < n:
                trmm("L", "L", "N", diag, 1.0, a[j1:, j1:], a[j1:, j0:j1], nb)
                trsm("R", "L", "N", diag, -1.0, a[j0:j1, j0:j1], a[j1:, j0:j1], nb)
            _trti2(a[j0:j1, j0:j1], True, unit, nb)
    return 0


def _lauu2(a, lower, herm):
    """Unblocked L^H L / U U^H (kernels.py:554-572)."""
    k = a.shape[0]
    if lower:
        for i in range(k):
            below = a[i + 1:, i].copy()
            aii = a[i, i]
            if i:
                r = (np.conj(aii) if herm else aii) * a[i, :i]
                if i + 1 < k:
                    r = r + (np.conj(below) if herm else below) @ a[i + 1:, :i]
                a[i, :i] = r
            d = np.vdot(below, below) + np.conj(aii) * aii
            a[i, i] = d.real if herm else d
    else:
        for j in range(k):
            row = np.conj(a[j, j:]) if herm else a[j, j:].copy()
            a[:j + 1, j] = a[:j + 1, j:] @ row
            if herm:
                a[j, j] = a[j, j].real


def lauum(uplo, a, nb=None):
    """Blocked in-place L^H L (lower) / U U^H (upper) (kernels.py:575-606)."""
    nb = NB if nb is None else nb
    n = a.shape[0]
    herm = np.iscomplexobj(a)
    for i0 in range(0, n, nb):
        i1 = min(n, i0 + nb)
        blk = a[i0:i1, i0:i1]
        if uplo == "L":
            if i0:
                trmm("L", "L", "C", "N", 1.0, blk, a[i0:i1, :i0], nb)
                if i1 < n:
                    gemm("C", "N", 1.0, a[i1:, i0:i1], a[i1:, :i0], 1.0, a[i0:i1, :i0])
            _lauu2(blk, True, herm)
            if i1 < n:
                syrk_herk("L", "C", 1.0, a[i1:, i0:i1], 1.0, blk, herm)
        else:
            if i0:
                trmm("R", "U", "C", "N", 1.0, blk, a[:i0, i0:i1], nb)
                if i1 < n:
                    gemm("N", "C", 1.0, a[:i0, i1:], a[i0:i1, i1:], 1.0, a[:i0, i0:i1])
            _lauu2(blk, False, herm)
            if i1 < n:
                syrk_herk("U", "N", 1.0, a[i0:i1, i1:], 1.0, blk, herm)


# ---------------------------------------------------------------------------
# RFP algorithms (rfp.py:55-360)


def pftrf(buf, n, uplo, transr):
    """SRPA factorization in place on the flat buffer (rfp.py:55-91)."""
    ds = desc(n, uplo, transr)
    if n == 0:
        return 0
    herm = np.iscomplexobj(buf)
    t1, t2, s1 = blocks(buf, ds)
    if ds.uplo == "L":
        info = potrf("L", t1)
        if info:
            return info
        if ds.n2:
            trsm("R", "L", "C", "N", 1.0, t1, s1)
            syrk_herk("U", "C", -1.0, s1.T, 1.0, t2, herm)
            info = potrf("U", t2)
            if info:
                return ds.n1 + info
        return 0
    if ds.n2:
        info = potrf("L", t1)
        if info:
            return info
        trsm("L", "U", "C", "N", 1.0, t1.T, s1)
        syrk_herk("U", "C", -1.0, s1, 1.0, t2, herm)
    info = potrf("U", t2)
    return ds.n2 + info if info else 0


def pftrs(buf, n, uplo, transr, b):
    """Forward/back substitution through T1/S1/T2, in place on b
    (rfp.py:106-136)."""
    ds = desc(n, uplo, transr)
    bv = b.reshape(-1, 1) if b.ndim == 1 else b
    if n == 0 or bv.shape[1] == 0:
        return
    t1, t2, s1 = blocks(buf, ds)
    n1, n2 = ds.n1, ds.n2
    if ds.uplo == "L":
        b1, b2 = bv[:n1], bv[n1:]
        trsm("L", "L", "N", "N", 1.0, t1, b1)
        if n2:
            gemm("N", "N", -1.0, s1, b1, 1.0, b2)
            trsm("L", "U", "T", "N", 1.0, t2, b2)
            trsm("L", "L", "C", "N", 1.0, t2.T, b2)
            gemm("C", "N", -1.0, s1, b2, 1.0, b1)
        trsm("L", "L", "C", "N", 1.0, t1, b1)
    else:
        b1, b2 = bv[:n2], bv[n2:]
        if n2:
            trsm("L", "U", "C", "N", 1.0, t1.T, b1)
            gemm("C", "N", -1.0, s1, b1, 1.0, b2)
        trsm("L", "U", "C", "N", 1.0, t2, b2)
        trsm("L", "U", "N", "N", 1.0, t2, b2)
        if n2:
            gemm("N", "N", -1.0, s1, b2, 1.0, b1)
            trsm("L", "L", "T", "N", 1.0, t1, b1)


def tftri(buf, n, uplo, transr, diag="N"):
    """Triangular inverse in RFP (rfp.py:286-325)."""
    ds = desc(n, uplo, transr)
    if n == 0:
        return 0
    t1, t2, s1 = blocks(buf, ds)
    n1, n2 = ds.n1, ds.n2
    if ds.uplo == "L":
        info = trtri("L", diag, t1)
        if info:
            return info
        if n2:
            trmm("R", "L", "N", diag, -1.0, t1, s1)
            info = trtri("U", diag, t2)
            if info:
                return n1 + info
            trmm("L", "U", "T", diag, 1.0, t2, s1)
        return 0
    if n2:
        info = trtri("L", diag, t1)
        if info:
            return info
        trmm("L", "L", "T", diag, -1.0, t1, s1)
        info = trtri("U", diag, t2)
        if info:
            return n2 + info
        trmm("R", "U", "N", diag, 1.0, t2, s1)
        return 0
    return trtri("U", diag, t2)


def pftri(buf, n, uplo, transr):
    """tftri then the lauum stage (rfp.py:328-360)."""
    info = tftri(buf, n, uplo, transr, "N")
    if info or n == 0:
        return info
    ds = desc(n, uplo, transr)
    herm = np.iscomplexobj(buf)
    t1, t2, s1 = blocks(buf, ds)
    if ds.uplo == "L":
        lauum("L", t1)
        if ds.n2:
            syrk_herk("L", "C", 1.0, s1, 1.0, t1, herm)
            trmm("L", "L", "C", "N", 1.0, t2.T, s1)
            lauum("U", t2)
    else:
        if ds.n2:
            lauum("L", t1)
            syrk_herk("L", "C", 1.0, s1.T, 1.0, t1, herm)
            trmm("R", "U", "C", "N", 1.0, t2, s1)
        lauum("U", t2)
    return 0


# ---------------------------------------------------------------------------
# SURVEY 8(f) "next" rows: tfsm, sfrk_hfrk, lansf (rfp.py:139-417)


def _tfsm_left(buf, ds, uplo, trans, diag, alpha, b):
    """Left RFP triangular solve through T1/S1/T2 (rfp.py:139-178); singular
    indices re-based to the global row (rfp.py:46-52)."""
    n1, n2 = ds.n1, ds.n2
    t1, t2, s1 = blocks(buf, ds)

    def solve(base, *args):
        try:
            trsm(*args)
        except OracleSingular as exc:
            raise OracleSingular(base + exc.index) from None

    if uplo == "L":
        b1, b2 = b[:n1], b[n1:]
        if trans == "N":
            solve(0, "L", "L", "N", diag, alpha, t1, b1)
            if n2:
                gemm("N", "N", -1.0, s1, b1, alpha, b2)
                solve(n1, "L", "U", "T", diag, 1.0, t2, b2)
        elif trans == "T":
            if n2:
                solve(n1, "L", "U", "N", diag, alpha, t2, b2)
                gemm("T", "N", -1.0, s1, b2, alpha, b1)
                solve(0, "L", "L", "T", diag, 1.0, t1, b1)
            else:
                solve(0, "L", "L", "T", diag, alpha, t1, b1)
        else:
            if n2:
                solve(n1, "L", "L", "C", diag, alpha, t2.T, b2)
                gemm("C", "N", -1.0, s1, b2, alpha, b1)
                solve(0, "L", "L", "C", diag, 1.0, t1, b1)
            else:
                solve(0, "L", "L", "C", diag, alpha, t1, b1)
    else:
        b1, b2 = b[:n2], b[n2:]
        if trans == "N":
            solve(n2, "L", "U", "N", diag, alpha, t2, b2)
            if n2:
                gemm("N", "N", -1.0, s1, b2, alpha, b1)
                solve(0, "L", "L", "T", diag, 1.0, t1, b1)
        elif trans == "T":
            if n2:
                solve(0, "L", "L", "N", diag, alpha, t1, b1)
                gemm("T", "N", -1.0, s1, b1, alpha, b2)
                solve(n2, "L", "U", "T", diag, 1.0, t2, b2)
            else:
                solve(n2, "L", "U", "T", diag, alpha, t2, b2)
        else:
            if n2:
                solve(0, "L", "U", "C", diag, alpha, t1.T, b1)
                gemm("C", "N", -1.0, s1, b1, alpha, b2)
                solve(n2, "L", "U", "C", diag, 1.0, t2, b2)
            else:
                solve(n2, "L", "U", "C", diag, alpha, t2, b2)


def tfsm(buf, nord, uplo, transr, side, trans, diag, alpha, b):
    """op(A) X = alpha B (side L) / X op(A) = alpha B (side R) with an
    RFP-stored triangle of order ``nord`` (rfp.py:181-224); in place on b."""
    ds = desc(nord, uplo, transr)
    m, n = b.shape
    if m == 0 or n == 0:
        return
    if alpha == 0:
        b[...] = 0
        return
    if not np.iscomplexobj(buf) and trans == "C":
        trans = "T"
    if side == "L":
        _tfsm_left(buf, ds, uplo, trans, diag, alpha, b)
    elif trans == "C":
        np.conjugate(b, out=b)
        _tfsm_left(buf, ds, uplo, "N", diag, np.conj(alpha), b.T)
        np.conjugate(b, out=b)
    else:
        _tfsm_left(buf, ds, uplo, "T" if trans == "N" else "N", diag, alpha, b.T)


def sfrk_hfrk(buf, n, uplo, transr, trans, k, alpha, a, beta, herm):
    """C <- alpha G G^(T|H) + beta C on an RFP triangle (rfp.py:227-283)."""
    ds = desc(n, uplo, transr)
    if n == 0:
        return
    if alpha == 0 or k == 0:
        if beta == 0:
            buf[...] = 0
        elif beta != 1:
            buf *= beta
        return
    n1, n2 = ds.n1, ds.n2
    t1, t2, s1 = blocks(buf, ds)
    rows = trans == "N"
    if ds.uplo == "L":
        a1 = a[:n1, :] if rows else a[:, :n1]
        a2 = a[n1:, :] if rows else a[:, n1:]
        syrk_herk("L", trans, alpha, a1, beta, t1, herm)
        if n2:
            gemm("N", "C", alpha, a2, a1, beta, s1) if rows else gemm("C", "N", alpha, a2, a1, beta, s1)
            syrk_herk("U", "C" if rows else "N", alpha, a2.T, beta, t2, herm)
    else:
        a1 = a[:n2, :] if rows else a[:, :n2]
        a2 = a[n2:, :] if rows else a[:, n2:]
        if n2:
            syrk_herk("L", "C" if rows else "N", alpha, a1.T, beta, t1, herm)
            gemm("N", "C", alpha, a1, a2, beta, s1) if rows else gemm("C", "N", alpha, a1, a2, beta, s1)
        syrk_herk("U", trans, alpha, a2, beta, t2, herm)


def lansf(norm, buf, n, uplo, transr):
    """Norm of the implied full symmetric/Hermitian matrix (rfp.py:363-417):
    'M' max |a|, '1'/'O'/'I' max column |.|-sum, 'F'/'E' Frobenius."""
    norm = str(norm).upper()[:1]
    if n == 0:
        return 0.0
    if norm == "M":
        return float(np.abs(buf).max())
    full = expand_hermitian(buf, n, uplo, transr)
    if norm in ("1", "O", "I"):
        return float(np.abs(full).sum(axis=0).max())
    return float(np.sqrt((np.abs(full) ** 2).sum()))


# ---------------------------------------------------------------------------
# seeded inputs (BASELINE.json configs; RNG convention of packed.py:166)


def spd_matrix(n, seed, scale="n", complex_=False):
    """A = B B^H + n I (scale='n', configs 1,2,4) or B B^H / n + I
    (scale='1/n', configs 3,5); B ~ N(0,1) real or N(0,1/2)+iN(0,1/2)."""
    rng = np.random.default_rng(seed)
    if complex_:
        s = np.sqrt(0.5)
        bm = rng.standard_normal((n, n)) * s + 1j * (rng.standard_normal((n, n)) * s)
    else:
        bm = rng.standard_normal((n, n))
    if scale == "n":
        a = bm @ np.conj(bm.T) + n * np.eye(n)
    else:
        a = bm @ np.conj(bm.T) / n + np.eye(n)
    return np.asfortranarray(a)


def expand_hermitian(buf, n, uplo, transr):
    """The full symmetric/Hermitian matrix implied by an RFP buffer."""
    t = tfttr(buf, n, uplo, transr)
    off = np.tril(t, -1) if uplo == "L" else np.triu(t, 1)
    return t + np.conj(off.T)


def expand_triangular(buf, n, uplo, transr):
    """The triangular factor implied by an RFP buffer (L or U)."""
    return tfttr(buf, n, uplo, transr)
