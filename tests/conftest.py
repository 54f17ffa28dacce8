import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden", "golden.npz")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built extension")
    config.addinivalue_line("markers", "slow: long-running (full BASELINE sizes)")


@pytest.fixture(scope="session")
def golden():
    with np.load(GOLDEN) as z:
        return {k: z[k] for k in z.files}


def golden_cases(g):
    """(key, dtype, uplo, transr, n) for every golden SPD case."""
    out = []
    for k in g:
        if k.endswith("_rfp") and not k.startswith(("fail_", "spec_", "lansf_", "tfsm_", "sfrk_")):
            base = k[:-4]
            dt, ut, nn = base.split("_")
            out.append((base, dt, ut[0], ut[1], int(nn[1:])))
    return sorted(out)


def next_row_cases(g):
    """(key, dtype, uplo, transr, n) for the SURVEY 8(f) golden cases."""
    out = []
    for k in g:
        if k.startswith("lansf_") and k.endswith("_rfp"):
            base = k[len("lansf_"):-4]
            dt, ut, nn = base.split("_")
            out.append((base, dt, ut[0], ut[1], int(nn[1:])))
    return sorted(out)
