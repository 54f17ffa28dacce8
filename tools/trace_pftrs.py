import os, sys, torch
os.environ["RFPK_TRACE"] = "1"; os.environ["RFPK_GRAPHS"] = "0"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__))); sys.path.insert(0, ROOT)
from paper_0901_1696_b200 import _capi, convert
lib = _capi.lib(); dev = torch.device("cuda:0"); st = _capi.stream_handle(dev)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
nrhs = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
g = torch.randn(n, n, dtype=torch.float64, device=dev); a = g @ g.t() / n; a.diagonal().add_(1.0)
r = convert.trttf(a, "L", "N"); del a, g
info = torch.zeros(1, dtype=torch.int32, device=dev)
lib.rfpk_dpftrf(b"N", b"L", n, r.data.data_ptr(), info.data_ptr(), st)
b0 = torch.randn(nrhs, n, dtype=torch.float64, device=dev).t(); b = b0.clone()
for rep in range(2):
    b.copy_(b0); torch.cuda.synchronize(); print("rep", rep, file=sys.stderr, flush=True)
    lib.rfpk_dpftrs(b"N", b"L", n, nrhs, r.data.data_ptr(), b.data_ptr(), n, info.data_ptr(), st)
    torch.cuda.synchronize()
