"""Phase and kernel timeline of one RFP call through the library's phase
clock (rfpk_phase_clock: CUDA event pairs on the launching streams around
every SRPA step and every kernel launch; no nsys here).

  python tools/trace.py pftrf|pftrs|pfsv|pftri n [uplo transr d|z nrhs]
"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_0901_1696_b200 import _capi, convert, rfp  # noqa: E402


def main():
    op, n = sys.argv[1], int(sys.argv[2])
    uplo = sys.argv[3] if len(sys.argv) > 3 else "L"
    transr = sys.argv[4] if len(sys.argv) > 4 else "N"
    cplx = len(sys.argv) > 5 and sys.argv[5] == "z"
    nrhs = int(sys.argv[6]) if len(sys.argv) > 6 else 1024
    dt = torch.complex128 if cplx else torch.float64
    g = torch.Generator(device="cuda").manual_seed(n)
    b = torch.randn(n, n, dtype=dt, device="cuda", generator=g)
    a = b @ b.mH / n
    a.diagonal().add_(1.0)
    del b
    r = convert.trttf(a, uplo, transr)
    x = torch.randn(nrhs, n, dtype=dt, device="cuda", generator=g).t()
    with _capi.tuning(graphs=0):
        if op in ("pftrs", "pftri"):
            assert rfp.pftrf(r) == 0
        torch.cuda.synchronize()
        with _capi.phase_clock() as pc:
            if op == "pftrf":
                assert rfp.pftrf(r) == 0
            elif op == "pftrs":
                rfp.pftrs(r, x)
            elif op == "pfsv":
                assert rfp.pfsv(r, x) == 0
            else:
                assert rfp.pftri(r) == 0
            torch.cuda.synchronize()
    for lab, (ms, cnt) in sorted(pc.table().items(), key=lambda kv: -kv[1][0]):
        print(f"{ms:10.3f} ms  x{cnt:<4d} {lab}")


if __name__ == "__main__":
    main()
