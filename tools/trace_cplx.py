"""Phase trace of complex pftrf (TRANSR='C', UPLO='L') at n (argv)."""
import os, sys, torch
os.environ["RFPK_TRACE"] = "1"; os.environ["RFPK_GRAPHS"] = "0"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__))); sys.path.insert(0, ROOT)
from paper_0901_1696_b200 import _capi, convert
lib = _capi.lib(); dev = torch.device("cuda:0"); st = _capi.stream_handle(dev)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 12000
g = torch.randn(n, n, dtype=torch.complex128, device=dev); a = g @ g.mH / n; a.diagonal().add_(1.0)
r = convert.trttf(a, "L", "C"); d0 = r.data.clone(); info = torch.zeros(1, dtype=torch.int32, device=dev)
del a, g
for rep in range(2):
    r.data.copy_(d0); torch.cuda.synchronize()
    print(f"n={n} rep={rep}", file=sys.stderr, flush=True)
    lib.rfpk_zpftrf(b"C", b"L", n, r.data.data_ptr(), info.data_ptr(), st)
    torch.cuda.synchronize()
