"""Utilisation over time of the dataflow tile trsm (RFPK_TILE_TRACE stamps)
for pftrs at (n, nrhs).  usage: trsm_trace.py n nrhs"""
import os, sys, tempfile
import numpy as np
n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
nrhs = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
trace = os.path.join(tempfile.mkdtemp(), "trace.csv")
os.environ["RFPK_GRAPHS"] = "0"
os.environ["RFPK_TILE_TRACE"] = trace
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__))); sys.path.insert(0, ROOT)
import torch
from paper_0901_1696_b200 import _capi, convert
lib = _capi.lib(); dev = torch.device("cuda:0"); st = _capi.stream_handle(dev)
g = torch.randn(n, n, dtype=torch.float64, device=dev); a = g @ g.t() / n; a.diagonal().add_(1.0)
r = convert.trttf(a, "L", "N"); del a, g
info = torch.zeros(1, dtype=torch.int32, device=dev)
lib.rfpk_dpftrf(b"N", b"L", n, r.data.data_ptr(), info.data_ptr(), st)
b = torch.randn(nrhs, n, dtype=torch.float64, device=dev).t()
torch.cuda.synchronize()
open(trace, "w").close()  # keep only the pftrs launches
lib.rfpk_dpftrs(b"N", b"L", n, nrhs, r.data.data_ptr(), b.data_ptr(), n, info.data_ptr(), st)
torch.cuda.synchronize()
blocks, cur = [], None
for l in open(trace):
    if l.startswith("#"):
        cur = [] if l.startswith("# trsm") else None
        if cur is not None:
            blocks.append((l.strip(), cur))
        continue
    if cur is not None:
        cur.append(list(map(int, l.split(","))))
for hdr, rows in blocks:
    # i, c, cta, t0, t1(acc done), t2, t3(published)
    t00 = min(x[3] for x in rows); tend = max(x[6] for x in rows)
    ctas = len({x[2] for x in rows})
    busy = sum(x[6] - x[3] for x in rows)
    print(hdr, "span %.0f us, CTAs %d, utilisation %.1f%%" % ((tend - t00) / 1e3, ctas, 100.0 * busy / ((tend - t00) * ctas)))
    edges = np.linspace(t00, tend, 11)
    print("   " + " ".join("%3.0f" % (100.0 * sum(max(0, min(x[6], e1) - max(x[3], e0)) for x in rows) / ((e1 - e0) * ctas))
                          for e0, e1 in zip(edges[:-1], edges[1:])))

# chain breakdown per column block c: previous step published -> this task's
# accumulation done (flag detection + last chunk + its GEMM) -> published
for hdr, rows in blocks[:1]:
    by = {(x[0], x[1]): x for x in rows}
    nb = 1 + max(x[0] for x in rows)
    steps = []
    for (i, c), x in by.items():
        p = by.get((i - 1, c))
        if p is None:
            continue
        steps.append(((x[4] - p[6]) / 1e3, (x[6] - x[4]) / 1e3, (x[6] - p[6]) / 1e3))
    if steps:
        a = np.array(steps)
        print("chain step (us): prev publish -> acc done %.2f | acc done -> publish %.2f | step %.2f"
              % tuple(a.mean(0)))
