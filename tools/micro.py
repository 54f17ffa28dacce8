"""Event-timed micro benchmarks of individual C-ABI kernels (developer tool)."""
import os, sys, json
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_0901_1696_b200 import _capi
lib = _capi.lib(); dev = torch.device("cuda:0"); st = lambda: _capi.stream_handle(dev)

def t(fn, reps=50):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    s.record()
    for _ in range(reps): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / reps * 1000  # us

info = torch.zeros(1, dtype=torch.int32, device=dev)
res = {}
for (m, n, k) in [(64, 64, 64), (64, 4096, 64), (4096, 64, 64), (128, 128, 128), (2000, 64, 2000), (256, 256, 256)]:
    a = torch.randn(k, m, dtype=torch.float64, device=dev).t()
    b = torch.randn(n, k, dtype=torch.float64, device=dev).t()
    c = torch.randn(n, m, dtype=torch.float64, device=dev).t()
    res[f"dgemm {m}x{n}x{k}"] = t(lambda: lib.rfpk_dgemm(b"N", b"N", -1.0, a.data_ptr(), m, k, 1, m, b.data_ptr(), k, n, 1, k, 1.0, c.data_ptr(), m, n, 1, m, st()))
for n in (64, 128, 256, 1024):
    g = torch.randn(n, n, dtype=torch.float64, device=dev); a0 = g @ g.t() + n * torch.eye(n, dtype=torch.float64, device=dev)
    a = a0.clone()
    res[f"dpotrf {n}"] = t(lambda: (a.copy_(a0), lib.rfpk_dpotrf(b"L", a.data_ptr(), n, 1, n, info.data_ptr(), st())), 20)
    res[f"copy {n}"] = t(lambda: a.copy_(a0), 20)
    l0 = torch.linalg.cholesky(a0); l = l0.clone()
    res[f"dtrtri {n}"] = t(lambda: (l.copy_(l0), lib.rfpk_dtrtri(b"L", b"N", l.data_ptr(), n, 1, n, info.data_ptr(), st())), 20)
    b = torch.randn(64, n, dtype=torch.float64, device=dev).t().contiguous().t()
    res[f"dtrsm {n} x64"] = t(lambda: lib.rfpk_dtrsm(b"L", b"L", b"N", b"N", 1.0, l0.data_ptr(), n, 1, n, b.data_ptr(), n, 64, 1, n, info.data_ptr(), st()), 20)
    res[f"dlauum {n}"] = t(lambda: (l.copy_(l0), lib.rfpk_dlauum(b"L", l.data_ptr(), n, 1, n, st())), 20)
for k, v in res.items():
    print(f"{v:10.1f} us  {k}")
