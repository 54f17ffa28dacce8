import os, sys, torch
sys.path.insert(0, os.getcwd())
from paper_0901_1696_b200 import _capi, convert
n = 24000
lib = _capi.lib(); dev = torch.device("cuda:0"); st = _capi.stream_handle(dev)
g = torch.randn(n, n, dtype=torch.complex128, device=dev)
a = g @ g.mH / n; a.diagonal().add_(1.0); del g
r = convert.trttf(a, "L", "C"); del a
info = torch.zeros(1, dtype=torch.int32, device=dev)
lib.rfpk_zpftrf(b"C", b"L", n, r.data.data_ptr(), info.data_ptr(), st)
fac = r.data.clone()
torch.cuda.synchronize()
_capi.set_tuning("trace", 1)
for rep in range(2):
    r.data.copy_(fac)
    torch.cuda.synchronize()
    lib.rfpk_zpftri(b"C", b"L", n, r.data.data_ptr(), info.data_ptr(), st)
    torch.cuda.synchronize()
print("info", int(info.item()))
