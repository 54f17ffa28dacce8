"""Time blas potrf (lower, column-major) for a range of n (CUDA events)."""
import os, sys, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__))); sys.path.insert(0, ROOT)
from paper_0901_1696_b200 import _capi
lib = _capi.lib(); dev = torch.device("cuda:0"); st = _capi.stream_handle(dev)
info = torch.zeros(1, dtype=torch.int32, device=dev)
UPLO = os.environ.get("UPLO", "L").encode()
for n in [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "500,1000,2000,4000,8192").split(",")]:
    g = torch.randn(n, n, dtype=torch.float64, device=dev); a = g @ g.t() / n; a.diagonal().add_(1.0)
    pad = int(os.environ.get("LDPAD", "0"))  # column stride n + pad (RFP blocks have odd ld)
    store = torch.zeros(n, n + pad, dtype=torch.float64, device=dev)
    w = store[:, :n]; ts = []
    for rep in range(6):
        w.copy_(a); torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); lib.rfpk_dpotrf(UPLO, w.data_ptr(), n, 1, n + pad, info.data_ptr(), st); e.record(); torch.cuda.synchronize()
        if rep >= 2: ts.append(s.elapsed_time(e))
    ms = sorted(ts)[len(ts) // 2]
    ref = torch.linalg.cholesky(a)  # w holds L column-major = L^T in torch row-major
    err = float((torch.triu(w).t() - ref).abs().max() / ref.abs().max())
    print(f"potrf n={n} {ms:.3f} ms {n**3/3/ms/1e9:.2f} TF info={int(info.item())} relerr={err:.1e}", flush=True)
    # cuSOLVER (torch) for reference
    ts = []
    for rep in range(5):
        torch.cuda.synchronize(); s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); torch.linalg.cholesky(a); e.record(); torch.cuda.synchronize()
        if rep >= 2: ts.append(s.elapsed_time(e))
    print(f"   cusolver n={n} {sorted(ts)[1]:.3f} ms", flush=True)
