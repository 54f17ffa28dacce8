import os, sys, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__))); sys.path.insert(0, ROOT)
from paper_0901_1696_b200 import _capi, convert
lib = _capi.lib(); dev = torch.device("cuda:0"); st = _capi.stream_handle(dev)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
g = torch.randn(n, n, dtype=torch.float64, device=dev); a = g @ g.t() / n; a.diagonal().add_(1.0)
r = convert.trttf(a, "L", "N"); d0 = r.data.clone(); info = torch.zeros(1, dtype=torch.int32, device=dev)
del a, g
ts = []
for rep in range(6):
    r.data.copy_(d0); torch.cuda.synchronize()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    s.record(); lib.rfpk_dpftrf(b"N", b"L", n, r.data.data_ptr(), info.data_ptr(), st); e.record()
    torch.cuda.synchronize(); ts.append(round(s.elapsed_time(e), 2))
print(os.environ.get("RFPK_GRAPHS", "1"), n, ts)
