"""pftrs-shaped solve (T1 of an n=16384 'N' 'L' RFP buffer, 1024 RHS) with the
right-hand side column-major (as pftrs receives it) vs row-major."""
import os, sys, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__))); sys.path.insert(0, ROOT)
from paper_0901_1696_b200 import _capi
from paper_0901_1696_b200.layout import make_descriptor
lib = _capi.lib(); dev = torch.device("cuda:0"); st = _capi.stream_handle(dev)
n = 16384; d = make_descriptor(n, "L", "N"); nrhs = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
buf = torch.randn(d.nt, dtype=torch.float64, device=dev) * 0.01
ld = d.ldar
k = torch.arange(d.n1, device=dev)
buf[d.shift + k + k * ld] = 4.0
t1 = buf.data_ptr() + 8 * d.shift
info = torch.zeros(1, dtype=torch.int32, device=dev)
for name, b in (("col-major", torch.randn(nrhs, d.n1, dtype=torch.float64, device=dev).t()),
                ("row-major", torch.randn(d.n1, nrhs, dtype=torch.float64, device=dev))):
    b0 = b.clone()
    def call():
        rc = lib.rfpk_dtrsm(b"L", b"L", b"N", b"N", 1.0, t1, d.n1, 1, ld, b.data_ptr(), d.n1, nrhs,
                            b.stride(0), b.stride(1), info.data_ptr(), st)
        assert rc == 0, rc
    call()
    ts = []
    for _ in range(3):
        b.copy_(b0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); call(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    ms = min(ts)
    print(f"{name}: {ms:.3f} ms  {d.n1 * d.n1 * nrhs / ms / 1e9:.2f} TFLOP/s")
