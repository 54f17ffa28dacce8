"""CTA utilisation over time of config 3's S1 solve (tile trsm, RFPK_TILE_TRACE)."""
import os, sys, tempfile
import numpy as np
trace = os.path.join(tempfile.mkdtemp(), "trace.csv")
os.environ["RFPK_TILE_TRACE"] = trace
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__))); sys.path.insert(0, ROOT)
import torch
from paper_0901_1696_b200 import _capi
from paper_0901_1696_b200.layout import make_descriptor
lib = _capi.lib(); dev = torch.device("cuda:0"); st = _capi.stream_handle(dev)
n = 16384; d = make_descriptor(n, "L", "N")
buf = torch.randn(d.nt, dtype=torch.float64, device=dev) * 0.01
ld = d.ldar
k = torch.arange(d.n1, device=dev)
buf[d.shift + k + k * ld] = 4.0
t1 = buf.data_ptr() + 8 * d.shift
s1 = buf.data_ptr() + 8 * (d.n1 + d.shift)
info = torch.zeros(1, dtype=torch.int32, device=dev)
lib.rfpk_dtrsm(b"R", b"L", b"C", b"N", 1.0, t1, d.n1, 1, ld, s1, d.n2, d.n1, 1, ld, info.data_ptr(), st)
torch.cuda.synchronize()
rows = [list(map(int, l.split(","))) for l in open(trace) if not l.startswith("#")]
t00 = min(x[3] for x in rows); tend = max(x[6] for x in rows)
ctas = len({x[2] for x in rows})
busy = sum(x[6] - x[3] for x in rows)
print("span %.0f us, CTAs %d, utilisation %.1f%%" % ((tend - t00) / 1e3, ctas, 100.0 * busy / ((tend - t00) * ctas)))
edges = np.linspace(t00, tend, 21)
print(" ".join("%3.0f" % (100.0 * sum(max(0, min(x[6], e1) - max(x[3], e0)) for x in rows) / ((e1 - e0) * ctas))
               for e0, e1 in zip(edges[:-1], edges[1:])))
