"""Per-matrix latency of the batched n=64 kernel without contention: batches of
148 (one warp per SM) .. 65,536 matrices, CUDA-event timed."""
import os, sys, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__))); sys.path.insert(0, ROOT)
from paper_0901_1696_b200 import _capi, convert
lib = _capi.lib(); dev = torch.device("cuda:0"); st = _capi.stream_handle(dev)
n, nrhs = 64, 8
g = torch.randn(n, n, dtype=torch.float64, device=dev); a = g @ g.t(); a.diagonal().add_(64.0)
one = convert.trttf(a, "U", "N").data
for batch in (148, 296, 148 * 4, 148 * 12, 148 * 48, 65536):
    arf0 = one.unsqueeze(0).repeat(batch, 1).contiguous()
    arf = arf0.clone()
    b0 = torch.randn(batch, nrhs, n, dtype=torch.float64, device=dev)
    b = b0.clone()
    info = torch.zeros(batch, dtype=torch.int32, device=dev)
    def restore():
        arf.copy_(arf0)
        b.copy_(b0)
    def call():
        lib.rfpk_dpftrf_pftrs_batched(b"N", b"U", n, nrhs, arf.data_ptr(), 2080, b.data_ptr(),
                                      n, n * nrhs, batch, info.data_ptr(), st)
    def timed(fn, reps=20):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(); e0.record()
        for _ in range(reps):
            fn()
        e1.record(); torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps
    for _ in range(3):
        restore(); call()
    ms = timed(lambda: (restore(), call())) - timed(restore)
    assert int(info.abs().sum()) == 0
    print(f"batch {batch:6d}: {ms*1e3:8.1f} us  {batch/ms*1e3/1e6:6.2f} M/s  "
          f"per-warp latency ~{ms*1e3*min(1.0, 148*12/batch):.1f} us")
