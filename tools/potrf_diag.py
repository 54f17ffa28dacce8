"""Which 64x64 tiles of a tile-potrf result are wrong (developer tool)."""
import os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_0901_1696_b200 import _capi
lib = _capi.lib(); dev = torch.device("cuda:0"); st = _capi.stream_handle(dev)
info = torch.zeros(1, dtype=torch.int32, device=dev)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
torch.manual_seed(n)
g = torch.randn(n, n, dtype=torch.float64, device=dev)
a = g @ g.t() / n; a.diagonal().add_(1.0)
ref = torch.linalg.cholesky(a)
for rep in range(2):
    w = a.clone(); info.zero_()
    lib.rfpk_dpotrf(b"L", w.data_ptr(), n, 1, n, info.data_ptr(), st); torch.cuda.synchronize()
    L = torch.tril(w.t())
    nt = (n + 63) // 64
    bad = []
    for J in range(nt):
        for I in range(J, nt):
            e = float((L[64*I:64*I+64, 64*J:64*J+64] - ref[64*I:64*I+64, 64*J:64*J+64]).abs().max())
            if e > 1e-10: bad.append((J, I, e))
    bad.sort()
    print(f"rep {rep}: info {int(info.item())}, {len(bad)} bad tiles; first (col, row, err):", bad[:8])
