"""Time one left-lower trsm (n x n, nrhs) through the C ABI; argv: n nrhs reps"""
import os, sys, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__))); sys.path.insert(0, ROOT)
from paper_0901_1696_b200 import _capi
lib = _capi.lib(); dev = torch.device("cuda:0"); st = _capi.stream_handle(dev)
n, nrhs, reps = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]) if len(sys.argv) > 3 else 5
info = torch.zeros(1, dtype=torch.int32, device=dev)
L = torch.randn(n, n, dtype=torch.float64, device=dev) / n ** 0.5; L.diagonal().add_(4.0)  # col-major via rs=1, cs=n
rowmajor = os.environ.get("BROW") == "1"
B0 = torch.randn(n, nrhs, dtype=torch.float64, device=dev) if rowmajor else \
    torch.randn(nrhs, n, dtype=torch.float64, device=dev)  # col-major n x nrhs
B = B0.clone(); ts = []
for r in range(reps):
    B.copy_(B0); torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    brs, bcs = (nrhs, 1) if rowmajor else (1, n)
    rc = lib.rfpk_dtrsm(b"L", b"L", b"N", b"N", 1.0, L.data_ptr(), n, 1, n, B.data_ptr(), n, nrhs, brs, bcs, info.data_ptr(), st)
    e.record(); torch.cuda.synchronize(); ts.append(s.elapsed_time(e))
ms = sorted(ts)[len(ts) // 2]
print(f"trsm n={n} nrhs={nrhs} rc={rc} {ms:.3f} ms {n*n*nrhs/ms/1e9:.2f} TF", flush=True)
