"""CPU-side checks of the C ABI: the shared library loads without a GPU and
exports every symbol include/rfpk_b200.h declares; the Python package mirrors
the reference's public names.  No compute calls (no GPU here)."""

import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "rfpk_b200.h")


def header_symbols():
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"\b(rfpk_\w+)\s*\(", txt)))


def test_header_and_binding_agree():
    from paper_0901_1696_b200 import _capi
    assert set(header_symbols()) == set(_capi.SIGNATURES)


def test_library_loads_and_exports_everything():
    from paper_0901_1696_b200 import _capi
    if not os.path.exists(_capi.LIB_PATH):
        pytest.skip("librfpk_b200.so not built (run __graft_entry__.build())")
    lib = _capi.load_library()
    for sym in header_symbols():
        assert hasattr(lib, sym), sym
    assert b"sm_100a" in lib.rfpk_version()


def test_no_cpu_fallback_without_device():
    import torch
    from paper_0901_1696_b200 import _capi
    if torch.cuda.is_available():
        pytest.skip("a device is present")
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        _capi.lib()
    from paper_0901_1696_b200 import convert
    with pytest.raises(RuntimeError):
        convert.trttf([[4.0, 0.0], [2.0, 5.0]], "L", "N")


def test_public_surface_mirrors_reference():
    import paper_0901_1696_b200 as P
    from paper_0901_1696_b200 import convert, kernels, layout, packed, rfp
    assert {"LayoutDescriptor", "BlockView", "make_descriptor", "map_index",
            "block_views"} <= set(layout.__all__)
    assert {"FactorState", "RfpTriangle", "PackedTriangle", "trttf", "tfttr", "tpttf",
            "tfttp"} <= set(convert.__all__)
    assert {"pftrf", "pftrs", "tftri", "pftri"} <= set(rfp.__all__)
    assert {"pack", "unpack"} <= set(packed.__all__)
    assert {"gemm", "trsm", "trmm", "syrk_herk", "potrf_ref", "trtri_ref", "lauum_ref",
            "SingularMatrixError"} <= set(kernels.__all__)
    assert P.__version__


def test_product_package_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_0901_1696_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in txt.replace("no CPU fallback", ""), f
