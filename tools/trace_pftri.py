"""RFPK_TRACE phase times of tftri + pftri (usage: trace_pftri.py n [L|U] [N|T])."""
import os, sys, torch
os.environ["RFPK_TRACE"] = "1"; os.environ["RFPK_GRAPHS"] = "0"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__))); sys.path.insert(0, ROOT)
from paper_0901_1696_b200 import _capi, convert
lib = _capi.lib(); dev = torch.device("cuda:0"); st = _capi.stream_handle(dev)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
uplo = sys.argv[2] if len(sys.argv) > 2 else "L"
transr = sys.argv[3] if len(sys.argv) > 3 else "N"
g = torch.randn(n, n, dtype=torch.float64, device=dev); a = g @ g.t() / n; a.diagonal().add_(1.0)
r = convert.trttf(a, uplo, transr); del a, g
info = torch.zeros(1, dtype=torch.int32, device=dev)
lib.rfpk_dpftrf(transr.encode(), uplo.encode(), n, r.data.data_ptr(), info.data_ptr(), st)
f = r.data.clone()
for rep in range(2):
    r.data.copy_(f); torch.cuda.synchronize(); print("rep", rep, file=sys.stderr, flush=True)
    lib.rfpk_dpftri(transr.encode(), uplo.encode(), n, r.data.data_ptr(), info.data_ptr(), st)
    torch.cuda.synchronize()
