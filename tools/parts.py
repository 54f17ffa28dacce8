"""Time the pieces of pftrf n=16384 LN individually (potrf 8192, trsm, syrk) via the C ABI."""
import os, sys, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__))); sys.path.insert(0, ROOT)
from paper_0901_1696_b200 import _capi
lib = _capi.lib(); dev = torch.device("cuda:0"); st = _capi.stream_handle(dev)
def t(fn, setup=None, reps=3):
    ts = []
    for i in range(reps + 1):
        if setup: setup()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(True), torch.cuda.Event(True)
        s.record(); fn(); e.record(); torch.cuda.synchronize()
        if i: ts.append(s.elapsed_time(e))
    return sorted(ts)[len(ts) // 2]
info = torch.zeros(1, dtype=torch.int32, device=dev)
for m in [int(x) for x in (sys.argv[1:] or ["8192", "4096", "2048", "1024", "512"])]:
    g = torch.randn(m, m, dtype=torch.float64, device=dev)
    a0 = g @ g.t() / m; a0.diagonal().add_(1.0)
    a = a0.clone()
    ms = t(lambda: lib.rfpk_dpotrf(b"L", a.data_ptr(), m, 1, m, info.data_ptr(), st), lambda: a.copy_(a0))
    print(f"potrf {m}: {ms:.3f} ms  {m**3/3/ms/1e9:.2f} TF")
    l = torch.linalg.cholesky(a0)
    b0 = torch.randn(m, m, dtype=torch.float64, device=dev); b = b0.clone()
    ms = t(lambda: lib.rfpk_dtrsm(b"R", b"L", b"C", b"N", 1.0, l.data_ptr(), m, 1, m, b.data_ptr(), m, m, 1, m, info.data_ptr(), st), lambda: b.copy_(b0))
    print(f"trsm  {m} x {m}: {ms:.3f} ms  {m**3/ms/1e9:.2f} TF")
    c = a0.clone()
    ms = t(lambda: lib.rfpk_dsyrk(b"L", b"N", -1.0, b0.data_ptr(), m, m, 1, m, 1.0, c.data_ptr(), m, 1, m, st))
    print(f"syrk  {m} k={m}: {ms:.3f} ms  {m**3/ms/1e9:.2f} TF")
    ms = t(lambda: torch.linalg.cholesky(a0))
    print(f"cusolver potrf {m}: {ms:.3f} ms  {m**3/3/ms/1e9:.2f} TF")
