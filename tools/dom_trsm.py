"""The dominant kernel of bench.py (config 3) after the tile rewrite: pftrf's
S1 <- S1 T1^-H, i.e. tile_trsm_kernel solving conj(T1) X = S1^T with 8192
right-hand sides on the RFP views of an n=16384 TRANSR='N' UPLO='L' buffer,
run through the C ABI (rfpk_dtrsm 'R','L','C','N') as pftrf issues it.
argv: reps.  For ncu --set full and for the bench roofline."""
import os, sys, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__))); sys.path.insert(0, ROOT)
from paper_0901_1696_b200 import _capi
from paper_0901_1696_b200.layout import make_descriptor
lib = _capi.lib(); dev = torch.device("cuda:0"); st = _capi.stream_handle(dev)
n = 16384; d = make_descriptor(n, "L", "N")
buf = torch.randn(d.nt, dtype=torch.float64, device=dev) * 0.01
ld = d.ldar
k = torch.arange(d.n1, device=dev)
buf[d.shift + k + k * ld] = 4.0             # well-conditioned T1 diagonal
t1 = buf.data_ptr() + 8 * d.shift           # rect[shift:, 0:n1]
s1 = buf.data_ptr() + 8 * (d.n1 + d.shift)  # rect[n1+shift:, 0:n1]
info = torch.zeros(1, dtype=torch.int32, device=dev)
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 2
def call():
    rc = lib.rfpk_dtrsm(b"R", b"L", b"C", b"N", 1.0, t1, d.n1, 1, ld, s1, d.n2, d.n1, 1, ld,
                        info.data_ptr(), st)
    assert rc == 0, rc
call()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize(); e0.record()
for _ in range(reps):
    call()
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / reps
print("ok", int(info.item()), "trsm %.3f ms  %.2f TFLOP/s" % (ms, d.n1 * d.n1 * d.n2 / ms / 1e9))
