"""Utilisation profile of one tile-trsm launch (developer tool; needs the
chain-trace build: tools/build_variant.sh trace -DRFPK_CHAIN_TRACE, run with
RFPK_LIB=build/variants/trace.so).  Per-task start/end stamps -> number of
tasks in flight over time, and where the time between the first start and
the last end goes.

  python tools/task_trace.py [n nrhs]"""
import ctypes, os, sys
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__))); sys.path.insert(0, ROOT)
from paper_0901_1696_b200 import _capi
lib = _capi.lib(); dev = torch.device("cuda:0"); st = _capi.stream_handle(dev)
info = torch.zeros(1, dtype=torch.int32, device=dev)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
m = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
g = torch.randn(n, n, dtype=torch.float64, device=dev) / n ** 0.5
L = (torch.tril(g) + 2 * torch.eye(n, dtype=torch.float64, device=dev)).t().contiguous().t()
b0 = torch.randn(m, n, dtype=torch.float64, device=dev).t()
b = b0.clone()
TT = 1 << 16
buf = (ctypes.c_ulonglong * (2 * TT))()
for rep in range(3):
    b.copy_(b0)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    lib.rfpk_dtrsm(b"L", b"L", b"N", b"N", 1.0, L.data_ptr(), n, 1, n, b.data_ptr(), n, m, 1, n,
                   info.data_ptr(), st)
    e1.record()
    torch.cuda.synchronize()
ms = e0.elapsed_time(e1)
lib.rfpk_task_trace_read(buf, 2 * TT)
t = np.array(buf, dtype=np.float64).reshape(TT, 2)
ntask = (n // 64) * ((m + 63) // 64 if m > 256 else (m + 15) // 16)
t = t[:ntask]
t0 = t[:, 0].min()
s, e = (t[:, 0] - t0) / 1e3, (t[:, 1] - t0) / 1e3
span = e.max()
print(f"trsm {n}x{m}: {ms:.3f} ms event-timed, {ntask} tasks, stamped span {span:.0f} us")
grid = np.linspace(0, span, 41)
act = [int(((s <= x) & (e > x)).sum()) for x in grid]
print("tasks in flight at 2.5% steps:", act)
dur = e - s
print(f"task duration us: mean {dur.mean():.1f}, p50 {np.median(dur):.1f}, max {dur.max():.1f}")
last = np.sort(e)
for q in (0.5, 0.9, 0.99, 1.0):
    print(f"  {int(q * 100)}% of tasks done by {last[int(q * (ntask - 1))]:.0f} us")
