"""The dominant kernel of bench.py (config 3): SYRK T2 <- T2 - S1 S1^T on the
RFP views of an n=16384 TRANSR='N' UPLO='L' buffer (ldar = 16385, odd), run
through the C ABI exactly as pftrf issues it.  For ncu --set full."""
import os, sys, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__))); sys.path.insert(0, ROOT)
from paper_0901_1696_b200 import _capi
from paper_0901_1696_b200.layout import make_descriptor
lib = _capi.lib(); dev = torch.device("cuda:0"); st = _capi.stream_handle(dev)
n = 16384; d = make_descriptor(n, "L", "N")
buf = torch.randn(d.nt, dtype=torch.float64, device=dev)
ld = d.ldar
t2 = buf.data_ptr()                       # rect[0:n2, 0:n2] (d = 1)
s1 = buf.data_ptr() + 8 * (d.n1 + d.shift)  # rect[n1+1:, 0:n1]
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 2
def call():
    rc = lib.rfpk_dsyrk(b"U", b"C", -1.0, s1, d.n2, d.n1, 1, ld, 1.0, t2, d.n2, 1, ld, st)
    assert rc == 0
call()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize(); e0.record()
for _ in range(reps):
    call()
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / reps
print("ok syrk %.3f ms  %.2f TFLOP/s" % (ms, d.n2 * d.n2 * d.n1 / ms / 1e9))
