"""RFP geometry: descriptor, element->offset bijection and block geometry.

Host-side integer arithmetic only (no device work); mirrors the public
surface of the reference ``rfpk.layout`` so callers can switch imports.

Reference behaviour followed (``/root/reference/pkg/src/rfpk/layout.py``):

* ``make_descriptor``           -> layout.py:103-124  (n1=ceil(n/2), ldar odd)
* ``LayoutDescriptor.shift``    -> layout.py:75-78    (d = 1 for even n)
* ``map_index`` / rect cell     -> layout.py:127-163  (1-based offsets)
* ``block_views``               -> layout.py:166-197
* flag normalisation            -> layout.py:34-38    (first letter, upper)

Deliberate extension: ``transr='C'`` is accepted as an alias of the
verbatim-transposed layout ``'T'`` (the reference rejects it at
layout.py:31; BASELINE config 5 names it).  The descriptor keeps the
canonical ``'T'`` so the geometry is identical.
"""

from __future__ import annotations

from dataclasses import dataclass

__all__ = [
    "LayoutDescriptor",
    "BlockView",
    "make_descriptor",
    "map_index",
    "block_views",
    "normalize_flag",
]

_TRANSR_ALIASES = {"N": "N", "T": "T", "C": "T"}


def normalize_flag(value, allowed, what: str) -> str:
    """First character, upper-cased; ``ValueError`` if not in ``allowed``."""
    f = str(value).upper()[:1]
    if f not in allowed:
        raise ValueError(f"{what} must be one of {tuple(allowed)}, got {value!r}")
    return f


@dataclass(frozen=True)
class LayoutDescriptor:
    """Geometry of one RFP triangle of order ``n``.

    ``n1 = ceil(n/2)``, ``n2 = n - n1``, ``nt = n(n+1)/2`` stored scalars,
    ``ldar`` = rows of the normal ``ldar x n1`` rectangle (odd for n >= 1).
    ``transr`` is ``'N'`` (buffer = column-major ``ldar x n1``) or ``'T'``
    (buffer = column-major ``n1 x ldar``, i.e. the rectangle transposed).
    """

    n: int
    n1: int
    n2: int
    nt: int
    ldar: int
    uplo: str
    transr: str

    @property
    def even(self) -> bool:
        return self.n % 2 == 0

    @property
    def shift(self) -> int:
        return int(self.n % 2 == 0)


@dataclass(frozen=True)
class BlockView:
    """One of T1/T2/S1 inside the stored rectangle (0-based offsets in the
    buffer's own orientation)."""

    kind: str
    row_offset: int
    col_offset: int
    rows: int
    cols: int
    triangle: str
    conjugated: bool


def make_descriptor(n: int, uplo: str, transr: str) -> LayoutDescriptor:
    """Descriptor for an order-``n`` RFP triangle (``n = 0`` allowed).

    >>> d = make_descriptor(7, "L", "N")
    >>> (d.n1, d.n2, d.nt, d.ldar)
    (4, 3, 28, 7)
    """
    n = int(n)
    if n < 0:
        raise ValueError(f"matrix order must be nonnegative, got {n}")
    u = normalize_flag(uplo, "LU", "uplo")
    t = str(transr).upper()[:1]
    if t not in _TRANSR_ALIASES:
        raise ValueError(f"transr must be one of ('N', 'T', 'C'), got {transr!r}")
    half = n - n // 2
    return LayoutDescriptor(n=n, n1=half, n2=n // 2, nt=(n * n + n) // 2,
                            ldar=n + 1 - (n & 1), uplo=u,
                            transr=_TRANSR_ALIASES[t])


def rect_cell(desc: LayoutDescriptor, i: int, j: int):
    """0-based cell ``(r, c)`` of the normal ``ldar x n1`` rectangle that
    holds 0-based triangle element ``(i, j)``."""
    n, n1, n2 = desc.n, desc.n1, desc.n2
    if not (0 <= i < n and 0 <= j < n):
        raise IndexError(f"indices ({i + 1}, {j + 1}) outside matrix of order {n}")
    if desc.uplo == "L":
        if j > i:
            raise IndexError(f"({i + 1}, {j + 1}) is not in the stored lower triangle")
        if j < n1:
            return i + desc.shift, j
        return j - n1, i - n1 + 1 - desc.shift
    if i > j:
        raise IndexError(f"({i + 1}, {j + 1}) is not in the stored upper triangle")
    if j >= n2:
        return i, j - n2
    return j + n2 + 1, i


def map_index(desc: LayoutDescriptor, i: int, j: int) -> int:
    """1-based buffer offset of the 1-based triangle element ``(i, j)``.

    >>> d = make_descriptor(7, "L", "N")
    >>> [map_index(d, 5, 5), map_index(d, 7, 4), map_index(d, 2, 1)]
    [8, 28, 2]
    """
    r, c = rect_cell(desc, int(i) - 1, int(j) - 1)
    off = c * desc.ldar + r if desc.transr == "N" else r * desc.n1 + c
    return off + 1


def block_views(desc: LayoutDescriptor):
    """``(T1, T2, S1)`` geometry; swapped row/col for the transposed layout."""
    if desc.n < 1:
        raise ValueError("block_views requires n >= 1")
    n1, n2, d = desc.n1, desc.n2, desc.shift
    if desc.uplo == "L":
        spec = (("T1", d, 0, n1, n1, "lower", False),
                ("T2", 0, 1 - d, n2, n2, "upper", True),
                ("S1", n1 + d, 0, n2, n1, "full", False))
    else:
        spec = (("T1", n2 + 1, 0, n2, n2, "lower", True),
                ("T2", n2, 0, n1, n1, "upper", False),
                ("S1", 0, 0, n2, n1, "full", False))
    flip = {"lower": "upper", "upper": "lower", "full": "full"}
    out = []
    for kind, r0, c0, rows, cols, tri, conj in spec:
        if desc.transr == "T":
            r0, c0, rows, cols, tri = c0, r0, cols, rows, flip[tri]
        out.append(BlockView(kind, r0, c0, rows, cols, tri, conj))
    return tuple(out)


def block_geometry(desc: LayoutDescriptor):
    """Flat-buffer geometry of T1/T2/S1 as ``(offset, rows, cols, rs, cs)``
    in the *normal* orientation (element (i, j) of the block lives at
    ``offset + i*rs + j*cs``).  This is the geometry the device kernels use;
    it equals the reference's ``_blocks(rect_normal())`` views
    (convert.py:142-153, 83-87)."""
    n1, n2, d = desc.n1, desc.n2, desc.shift
    if desc.transr == "N":
        rs, cs = 1, desc.ldar
    else:
        rs, cs = desc.n1, 1
    if desc.uplo == "L":
        t1, t2, s1 = (d, 0, n1, n1), (0, 1 - d, n2, n2), (n1 + d, 0, n2, n1)
    else:
        t1, t2, s1 = (n2 + 1, 0, n2, n2), (n2, 0, n1, n1), (0, 0, n2, n1)
    return tuple((r0 * rs + c0 * cs, rows, cols, rs, cs) for r0, c0, rows, cols in (t1, t2, s1))
