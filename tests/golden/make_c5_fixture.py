"""Config 5 at FULL size, run through the REFERENCE itself (build container
only: imports /root/reference).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_c5_fixture.py [n]

complex128 n=24000, TRANSR 'C' (the reference's verbatim 'T' layout), UPLO
'L', A = B Bᴴ·fl(1/n) + I with the exact-Gram B of ``tests/inputs.c5_b``:
reference ``convert.trttf`` -> ``rfp.pftrf`` -> ``rfp.pftri``, then the 256
inverse columns J = ``inputs.c5_columns(n)``.

Writes
* ``tests/golden/large/c5_n{n}_invcols.npy`` -- all 256 columns (n x 256,
  98 MB; git-ignored, travels to the GPU box with the working tree);
* ``tests/golden/c5_n{n}_fixture.npz`` -- committed: J, 512 fixed rows of
  every column, two whole columns, per-column 2-norms, the SHA-256 of A's RFP
  buffer (the GPU test recomputes it to prove identical input bits) and of
  the full column block, and the reference's timings.
"""

import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")
from rfpk import convert, layout, rfp  # noqa: E402
from tests import inputs  # noqa: E402
from scipy.linalg.blas import zherk  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 24000
    t0 = time.time()
    b = inputs.c5_b(n)
    # exactness check on a slab: integer Gram (int64, exact) vs FP64 product
    bi = np.rint(b[:64].real * inputs.QUANT).astype(np.int64), np.rint(b[:64].imag * inputs.QUANT).astype(np.int64)
    g_re = bi[0] @ bi[0].T + bi[1] @ bi[1].T
    g_im = bi[1] @ bi[0].T - bi[0] @ bi[1].T
    a = np.asfortranarray(zherk(1.0, b, lower=1))     # lower triangle of B Bᴴ (exact)
    del b
    blk = a[:64, :64]
    low = np.tril(np.ones((64, 64), bool))
    assert np.array_equal(blk.real[low] * inputs.QUANT ** 2, g_re[low].astype(np.float64))
    assert np.array_equal(blk.imag[low] * inputs.QUANT ** 2, g_im[low].astype(np.float64))
    a *= np.float64(1.0) / n
    a[np.diag_indices(n)] += 1.0
    gen_s = time.time() - t0
    r = convert.trttf(a, "L", "T")
    del a
    a_sha = hashlib.sha256(r.data.tobytes()).hexdigest()
    t = time.time()
    info = rfp.pftrf(r)
    t_f = time.time() - t
    assert info == 0, info
    t = time.time()
    info = rfp.pftri(r)
    t_i = time.time() - t
    assert info == 0, info
    full = convert.tfttr(r)                   # lower triangle of A^-1
    del r
    J = inputs.c5_columns(n)
    low = full[:, J]
    up = np.conj(full[J, :].T)
    rows = np.arange(n)[:, None]
    Y = np.where(rows >= J[None, :], low, up)
    del full, low, up
    os.makedirs(os.path.join(HERE, "large"), exist_ok=True)
    np.save(os.path.join(HERE, "large", f"c5_n{n}_invcols.npy"), Y)
    R = np.sort(np.random.default_rng(12).choice(n, 512, replace=False))
    meta = {"n": n, "transr": "C (reference 'T')", "uplo": "L",
            "recipe": "B = rint(N(0,1/2) * 2^12) / 2^12 (re, im), A = B B^H * fl(1/n) + I (exact Gram)",
            "reference_pftrf_s": t_f, "reference_pftri_s": t_i, "gen_s": gen_s,
            "cpu_count": os.cpu_count(), "numpy": np.__version__}
    np.savez(os.path.join(HERE, f"c5_n{n}_fixture.npz"), J=J, R=R, Y_rows=Y[R], Y_cols01=Y[:, :2],
             col_norms=np.linalg.norm(Y, axis=0), a_rfp_sha256=np.array(a_sha),
             y_sha256=np.array(hashlib.sha256(np.ascontiguousarray(Y).tobytes()).hexdigest()),
             meta=np.array(json.dumps(meta)))
    print(json.dumps(meta))


if __name__ == "__main__":
    main()
