import os, sys, torch
os.environ["RFPK_TRACE"] = "1"; os.environ["RFPK_GRAPHS"] = "0"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__))); sys.path.insert(0, ROOT)
from paper_0901_1696_b200 import _capi, convert
lib = _capi.lib(); dev = torch.device("cuda:0"); st = _capi.stream_handle(dev)
# args: n or n:uplo:transr
CASES = [(int(a.split(":")[0]),) + tuple(a.split(":")[1:3] or ("L", "N")) for a in sys.argv[1:]] or [(16384, "L", "N"), (4000, "L", "N"), (1000, "L", "N")]
for n, u, t in CASES:
    g = torch.randn(n, n, dtype=torch.float64, device=dev); a = g @ g.t() / n; a.diagonal().add_(1.0)
    r = convert.trttf(a, u, t); d0 = r.data.clone(); info = torch.zeros(1, dtype=torch.int32, device=dev)
    for rep in range(2):
        r.data.copy_(d0); torch.cuda.synchronize()
        print(f"n={n} rep={rep}", file=sys.stderr, flush=True)
        lib.rfpk_dpftrf(t.encode(), u.encode(), n, r.data.data_ptr(), info.data_ptr(), st)
        torch.cuda.synchronize()
