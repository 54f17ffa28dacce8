import os, sys, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__))); sys.path.insert(0, ROOT)
from paper_0901_1696_b200 import _capi
lib = _capi.lib(); dev = torch.device("cuda:0"); st = _capi.stream_handle(dev)
m, n, k = [int(x) for x in sys.argv[1:4]]
a = torch.randn(k, m, dtype=torch.float64, device=dev).t()
b = torch.randn(n, k, dtype=torch.float64, device=dev).t()
c = torch.randn(n, m, dtype=torch.float64, device=dev).t()
for _ in range(3):
    lib.rfpk_dgemm(b"N", b"N", -1.0, a.data_ptr(), m, k, 1, m, b.data_ptr(), k, n, 1, k, 1.0, c.data_ptr(), m, n, 1, m, st)
torch.cuda.synchronize(); print("ok")
