"""Config 3 (n=16384 LN, nrhs=1024): the SRPA phase times of the device
call (rfpk_dpfsv) beside those of the host-buffer call (rfp.pfsv_from_host),
from the library's phase clock -- where the end-to-end path loses time."""
import os, sys, time
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__))); sys.path.insert(0, ROOT)
from paper_0901_1696_b200 import _capi, convert, rfp
dev = torch.device("cuda:0")
n, m = 16384, 1024
g = torch.from_numpy(np.random.default_rng(3).standard_normal((n, n))).to(dev)
a = g @ g.t() / n
a.diagonal().add_(1.0)
del g
r0 = convert.trttf(a, "L", "N").data
del a
b0 = torch.randn(m, n, dtype=torch.float64, device=dev).t()
host_rfp = r0.cpu().pin_memory()
host_b = b0.t().contiguous().cpu().pin_memory()
out = torch.empty_like(host_b).pin_memory()
lib = _capi.lib()
st = torch.cuda.current_stream(dev).cuda_stream
info = torch.zeros(1, dtype=torch.int32, device=dev)
work = torch.empty_like(r0)
x = torch.empty((m, n), dtype=torch.float64, device=dev).t()

def dev_call():
    work.copy_(r0); x.copy_(b0)
    lib.rfpk_dpfsv(b"N", b"L", n, m, work.data_ptr(), x.data_ptr(), n, info.data_ptr(), st)

def host_call():
    rfp.pfsv_from_host(host_rfp, host_b.t(), n, "L", "N", out=out.t())

for name, fn in (("device", dev_call), ("host", host_call)):
    fn(); fn(); torch.cuda.synchronize()
    with _capi.phase_clock() as pc:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); t0 = time.perf_counter()
        fn()
        e1.record(); torch.cuda.synchronize(); t1 = time.perf_counter()
    print(f"== {name}: {e0.elapsed_time(e1):.2f} ms events, {1e3 * (t1 - t0):.2f} ms wall")
    for lab, (ms, cnt) in sorted(pc.table().items(), key=lambda kv: -kv[1][0])[:12]:
        print(f"   {ms:8.3f} ms  x{cnt:<3d} {lab}")
# raw PCIe rates on this box
big = torch.empty(host_rfp.numel(), dtype=torch.float64, device=dev)
torch.cuda.synchronize(); t0 = time.perf_counter(); big.copy_(host_rfp, non_blocking=True); torch.cuda.synchronize()
print(f"H2D {host_rfp.numel() * 8 / (time.perf_counter() - t0) / 1e9:.1f} GB/s")
torch.cuda.synchronize(); t0 = time.perf_counter(); host_rfp.copy_(big, non_blocking=True); torch.cuda.synchronize()
print(f"D2H {host_rfp.numel() * 8 / (time.perf_counter() - t0) / 1e9:.1f} GB/s")
