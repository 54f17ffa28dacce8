"""Time pftrs alone (device-resident factor and RHS) for A/B runs of the
solve variants: python tools/pftrs_ab.py n nrhs [uplo transr] -- env vars
(RFPK_NO_TRSM2, RFPK_TRSM2_PREW, ...) select the variant."""
import json, os, sys
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_0901_1696_b200 import _capi, convert

lib = _capi.lib()
dev = torch.device("cuda:0")
st = _capi.stream_handle(dev)
n, nrhs = int(sys.argv[1]), int(sys.argv[2])
uplo = sys.argv[3] if len(sys.argv) > 3 else "L"
transr = sys.argv[4] if len(sys.argv) > 4 else "N"
g = torch.randn(n, n, dtype=torch.float64, device=dev)
a = g @ g.t() / n
a.diagonal().add_(1.0)
r = convert.trttf(a, uplo, transr)
del a, g
info = torch.zeros(1, dtype=torch.int32, device=dev)
lib.rfpk_dpftrf(transr.encode(), uplo.encode(), n, r.data.data_ptr(), info.data_ptr(), st)
b0 = torch.randn(nrhs, n, dtype=torch.float64, device=dev).t()
b = b0.clone()
ts = []
for rep in range(7):
    b.copy_(b0)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    lib.rfpk_dpftrs(transr.encode(), uplo.encode(), n, nrhs, r.data.data_ptr(), b.data_ptr(), n,
                    info.data_ptr(), st)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
ts = sorted(ts[2:])
env = {k: v for k, v in os.environ.items() if k.startswith("RFPK_")}
print(json.dumps(dict(n=n, nrhs=nrhs, uplo=uplo, transr=transr, env=env, ms=ts[len(ts) // 2],
                      tflops=2 * n * n * nrhs / ts[len(ts) // 2] / 1e9)))
