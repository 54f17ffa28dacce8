"""Time complex blas potrf (lower) for a range of n."""
import os, sys, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__))); sys.path.insert(0, ROOT)
from paper_0901_1696_b200 import _capi
lib = _capi.lib(); dev = torch.device("cuda:0"); st = _capi.stream_handle(dev)
info = torch.zeros(1, dtype=torch.int32, device=dev)
if "ZSPLIT" in os.environ:  # tuning zpotrf_split_min (a huge value = never split)
    _capi.set_tuning("zpotrf_split_min", int(os.environ["ZSPLIT"]))
for n in [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "1000,3000,6000").split(",")]:
    g = torch.randn(n, n, dtype=torch.complex128, device=dev); a = g @ g.mH / n; a.diagonal().add_(1.0)
    pad = int(os.environ.get("LDPAD", "0"))
    store = torch.zeros(n, n + pad, dtype=torch.complex128, device=dev)
    w = store[:, :n]; ts = []
    for rep in range(5):
        w.copy_(a); torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); lib.rfpk_zpotrf(os.environ.get("UPLO", "L").encode(), w.data_ptr(), n, 1, n + pad, info.data_ptr(), st); e.record(); torch.cuda.synchronize()
        if rep >= 1: ts.append(s.elapsed_time(e))
    ms = sorted(ts)[len(ts) // 2]
    print(f"zpotrf n={n} {ms:.3f} ms {4*n**3/3/ms/1e9:.2f} TF info={int(info.item())}", flush=True)
