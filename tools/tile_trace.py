"""Critical-path breakdown of the dataflow tile potrf from its per-task
globaltimer stamps (RFPK_TILE_TRACE).  usage: tile_trace.py n"""
import os, sys, tempfile
import numpy as np
n = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
trace = os.path.join(tempfile.mkdtemp(), "trace.csv")
os.environ["RFPK_TILE_TRACE"] = trace
os.environ["RFPK_GRAPHS"] = "0"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__))); sys.path.insert(0, ROOT)
import torch
from paper_0901_1696_b200 import kernels as K
g = torch.randn(n, n, dtype=torch.float64, device="cuda")
a = g @ g.t() / n + torch.eye(n, dtype=torch.float64, device="cuda")
for rep in range(2):
    open(trace, "w").close()
    ad = a.clone()
    assert K.potrf_ref("L", ad) == 0
rows = [list(map(int, l.split(","))) for l in open(trace) if not l.startswith("#")]
# kind,a,b,cta,t0,t1(acc),t2(W ready),t3(published),t6(X published),t7(diag updated)
# kinds: 0 DIAG0, 1 SUPER, 2 NORMAL, 3 PARTIAL
kinds = sorted({r[0] for r in rows})
print("kinds", kinds, "tasks", len(rows))
t00 = min(r[4] for r in rows)
tend = max(r[7] for r in rows)
print("span %.1f us" % ((tend - t00) / 1e3))
for k in kinds:
    rs = [r for r in rows if r[0] == k]
    d = np.array([(r[7] - r[4]) / 1e3 for r in rs])
    print("kind %d: %d tasks, duration mean %.1f us max %.1f" % (k, len(rs), d.mean(), d.max()))
# chain: tasks with 8 stamps (super): phases
for k in kinds:
    rs = [r for r in rows if r[0] == k and r[8] and r[9]]
    if not rs:
        continue
    ph = np.array([[r[5] - r[4], r[6] - r[5], r[8] - r[6], r[9] - r[8], r[7] - r[9]] for r in rs]) / 1e3
    print("kind %d phases (us): acc %.1f | wait W %.1f | apply_w %.1f | diag update %.1f | leaf %.1f"
          % ((k,) + tuple(ph.mean(0))))
    st = sorted(rs, key=lambda r: r[2])
    gaps = [(st[i + 1][6] - st[i][7]) / 1e3 for i in range(len(st) - 1)]
    print("  W_j published -> next super sees it: mean %.1f us" % np.mean(gaps))

# utilisation: busy CTA-time / (span x CTAs), and over time in 10 slices
ctas = len({r[3] for r in rows})
busy = sum(r[7] - r[4] for r in rows)
span = tend - t00
print("CTAs %d  utilisation %.1f%%" % (ctas, 100.0 * busy / (span * ctas)))
edges = np.linspace(t00, tend, 11)
for s in range(10):
    a0, a1 = edges[s], edges[s + 1]
    b = sum(max(0, min(r[7], a1) - max(r[4], a0)) for r in rows)
    print("  slice %d: %.0f%% busy" % (s, 100.0 * b / ((a1 - a0) * ctas)))
