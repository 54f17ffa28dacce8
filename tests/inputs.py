"""Seeded BASELINE.json inputs shared by the parity tests, the fixture
generators and bench.py (test infrastructure; SURVEY §8(d) recipe:
``numpy.random.default_rng(seed).standard_normal``, A built once on the host
and the identical bits fed to the oracle and to the GPU).

Config 5's full-size fixture is produced in another process (and on another
machine) than the GPU run it pins, so its A must be reproducible bit for bit
wherever it is formed.  ``c5_b_slab`` therefore rounds the N(0, 1/2) entries
to the 2**-12 grid: every product of two entries is then an integer multiple
of 2**-24 below 2**29, and every partial sum of B·Bᴴ (n = 24000 terms) stays
below 2**53 · 2**-24, so the Gram matrix is EXACT in FP64 -- the same bits
from OpenBLAS on the host and cuBLAS on the device, whatever the summation
order.  The scale 1/n is applied as a multiplication by fl(1/n) on both
sides (a true division on one side and a reciprocal multiply on the other
would differ in the last bit)."""

import numpy as np

C5_SEED = 5
C5_SLAB = 2000
QUANT = 4096.0          # 2**12


def spd_host(n, seed, scale, cplx=False):
    """A = B Bᴴ + n I (scale 'n': configs 1, 2, 4) or B Bᴴ/n + I (scale '1/n':
    configs 3, 5) with B ~ N(0,1) (complex: N(0,1/2) + i N(0,1/2)); built on
    the host in FP64 (column-major)."""
    rng = np.random.default_rng(seed)
    if cplx:
        s = np.sqrt(0.5)
        b = rng.standard_normal((n, n)) * s + 1j * (rng.standard_normal((n, n)) * s)
    else:
        b = rng.standard_normal((n, n))
    a = b @ np.conj(b.T)
    del b
    if scale == "n":
        a[np.diag_indices(n)] += n
    else:
        a /= n
        a[np.diag_indices(n)] += 1.0
    return np.asfortranarray(a)


def rhs_host(n, nrhs, seed, cplx=False):
    rng = np.random.default_rng(seed + 1000)
    b = rng.standard_normal((n, nrhs))
    if cplx:
        b = b + 1j * rng.standard_normal((n, nrhs))
    return np.asfortranarray(b)


def c5_b_slab(rng, rows, n):
    """One row slab of config 5's B: N(0,1/2) real and imaginary parts, rounded
    to the 2**-12 grid (see the module docstring).  Slabs are drawn in order
    from ONE generator: real part then imaginary part per slab."""
    s = np.sqrt(0.5)
    re = np.rint(rng.standard_normal((rows, n)) * s * QUANT) / QUANT
    im = np.rint(rng.standard_normal((rows, n)) * s * QUANT) / QUANT
    return re + 1j * im


def c5_b(n, seed=C5_SEED):
    rng = np.random.default_rng(seed)
    out = np.empty((n, n), np.complex128)
    for r0 in range(0, n, C5_SLAB):
        r1 = min(n, r0 + C5_SLAB)
        out[r0:r1] = c5_b_slab(rng, r1 - r0, n)
    return out


def c5_columns(n, count=256, seed=11):
    """The 256 random inverse columns J checked at config 5."""
    return np.sort(np.random.default_rng(seed).choice(n, count, replace=False))
