"""Config 4 split: fused pftrf+pftrs vs pftrf alone vs pftrs alone (65,536 x n=64)."""
import os, sys, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__))); sys.path.insert(0, ROOT)
from paper_0901_1696_b200 import _capi, convert
lib = _capi.lib(); dev = torch.device("cuda:0"); st = _capi.stream_handle(dev)
n, nrhs, batch = 64, 8, 65536
g = torch.randn(n, n, dtype=torch.float64, device=dev); a = g @ g.t(); a.diagonal().add_(64.0)
one = convert.trttf(a, "U", "N").data
arf0 = one.unsqueeze(0).repeat(batch, 1).contiguous(); arf = arf0.clone()
b0 = torch.randn(batch, nrhs, n, dtype=torch.float64, device=dev); b = b0.clone()
info = torch.zeros(batch, dtype=torch.int32, device=dev)
fac = arf0.clone()
lib.rfpk_dpftrf_batched(b"N", b"U", n, fac.data_ptr(), 2080, batch, info.data_ptr(), st)
def timed(setup, fn, reps=10):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    tot = 0.0
    for _ in range(reps):
        setup(); e0.record(); fn(); e1.record(); torch.cuda.synchronize(); tot += e0.elapsed_time(e1)
    return tot / reps
rs = lambda: (arf.copy_(arf0), b.copy_(b0))
fused = timed(rs, lambda: lib.rfpk_dpftrf_pftrs_batched(b"N", b"U", n, nrhs, arf.data_ptr(), 2080, b.data_ptr(), n, n * nrhs, batch, info.data_ptr(), st))
fonly = timed(rs, lambda: lib.rfpk_dpftrf_batched(b"N", b"U", n, arf.data_ptr(), 2080, batch, info.data_ptr(), st))
sonly = timed(rs, lambda: lib.rfpk_dpftrs_batched(b"N", b"U", n, nrhs, fac.data_ptr(), 2080, b.data_ptr(), n, n * nrhs, batch, info.data_ptr(), st))
print(f"fused {fused*1e3:.0f} us  pftrf only {fonly*1e3:.0f} us  pftrs only (incl. both inverses) {sonly*1e3:.0f} us")
