import os, sys, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__))); sys.path.insert(0, ROOT)
from paper_0901_1696_b200 import _capi, convert
lib = _capi.lib(); dev = torch.device("cuda:0"); st = _capi.stream_handle(dev)
batch, n, nrhs = int(sys.argv[1]) if len(sys.argv) > 1 else 65536, 64, 8
g = torch.randn(n, n, dtype=torch.float64, device=dev); a = g @ g.t(); a.diagonal().add_(64.0)
one = convert.trttf(a, "U", "N").data
arf = one.unsqueeze(0).repeat(batch, 1).contiguous()
b = torch.randn(batch, nrhs, n, dtype=torch.float64, device=dev)
info = torch.zeros(batch, dtype=torch.int32, device=dev)
for _ in range(2):
    lib.rfpk_dpftrf_pftrs_batched(b"N", b"U", n, nrhs, arf.data_ptr(), 2080, b.data_ptr(), n, n * nrhs, batch, info.data_ptr(), st)
torch.cuda.synchronize(); print("ok", int(info.abs().sum()))
