"""A/B of the tile trsm's split (PRE) tasks: rfpk_dtrsm on an 8192-order lower
triangle with 1024 right-hand sides (pftrs's solves of config 3), forward and
transposed, column-major B; tuning "trsm_split" = 0 / 16 / 24 / 32 / 48.

  python tools/trsm_split_ab.py [n nrhs]"""
import os, sys
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__))); sys.path.insert(0, ROOT)
from paper_0901_1696_b200 import _capi
lib = _capi.lib(); dev = torch.device("cuda:0"); st = _capi.stream_handle(dev)
info = torch.zeros(1, dtype=torch.int32, device=dev)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
m = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
torch.manual_seed(1)
g = torch.randn(n, n, dtype=torch.float64, device=dev) / n ** 0.5
L = (torch.tril(g) + 2 * torch.eye(n, dtype=torch.float64, device=dev)).t().contiguous().t()
ROWMAJOR = len(sys.argv) > 3 and sys.argv[3] == "row"
b0 = torch.randn(n, m, dtype=torch.float64, device=dev) if ROWMAJOR else \
    torch.randn(m, n, dtype=torch.float64, device=dev).t()
rsb, csb = (m, 1) if ROWMAJOR else (1, n)
ref = {}
for split in (0, 1, 16, 24, 32, 40):
    _capi.set_tuning("trsm_split", split)
    for trans in (b"N", b"T"):
        b = b0.clone()
        ts = []
        for rep in range(6):
            b.copy_(b0)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            rc = lib.rfpk_dtrsm(b"L", b"L", trans, b"N", 1.0, L.data_ptr(), n, 1, n, b.data_ptr(),
                                n, m, rsb, csb, info.data_ptr(), st)
            e1.record()
            torch.cuda.synchronize()
            assert rc == 0
            ts.append(e0.elapsed_time(e1))
        key = trans
        if split == 0:
            ref[key] = b.clone()
            err = 0.0
        else:
            err = float((b - ref[key]).abs().max() / ref[key].abs().max())
        print(f"split {split:2d} trans {trans.decode()}: {sorted(ts)[len(ts)//2]:.3f} ms  (min {min(ts):.3f})"
              f"  max rel diff vs unsplit {err:.2e}")
