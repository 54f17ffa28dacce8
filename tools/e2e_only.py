"""Time rfp.pfsv_from_host (the bench e2e path) for config 3; argv: reps."""
import os, sys, time, numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__))); sys.path.insert(0, ROOT)
from paper_0901_1696_b200 import convert, rfp
n, nrhs = 16384, 1024
dev = torch.device("cuda:0")
g = torch.randn(n, n, dtype=torch.float64, device=dev); a = g @ g.t() / n; a.diagonal().add_(1.0); del g
host_rfp = convert.trttf(a, "L", "N").data.cpu().pin_memory(); del a
host_b = torch.randn(nrhs, n, dtype=torch.float64).pin_memory()
out = torch.empty_like(host_b).pin_memory()
ts = []
for r in range(int(sys.argv[1]) if len(sys.argv) > 1 else 4):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    rr, inf = rfp.pfsv_from_host(host_rfp, host_b.t(), n, "L", "N", out=out.t())
    torch.cuda.synchronize(); ts.append((time.perf_counter() - t0) * 1e3)
    del rr
print("e2e ms", [round(x, 2) for x in ts], "median", sorted(ts)[len(ts) // 2], flush=True)
