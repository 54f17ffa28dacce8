import os, sys, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__))); sys.path.insert(0, ROOT)
from paper_0901_1696_b200 import _capi
lib = _capi.lib(); dev = torch.device("cuda:0"); st = _capi.stream_handle(dev)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
norm = (sys.argv[2] if len(sys.argv) > 2 else "1").encode()
tr = (sys.argv[3] if len(sys.argv) > 3 else "N").encode()
nt = n * (n + 1) // 2
arf = torch.randn(nt, dtype=torch.float64, device=dev)
res = torch.zeros(1, dtype=torch.float64, device=dev)
for _ in range(2):
    lib.rfpk_dlansf(norm, tr, b"L", n, arf.data_ptr(), res.data_ptr(), st)
torch.cuda.synchronize(); print("ok", float(res))
