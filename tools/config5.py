"""BASELINE config 5 at full size: complex128 n=24000, TRANSR='C' (== 'T'),
UPLO='L', A = B B^H / n + I (B re/im ~ N(0,1/2), seeded on the host), pftrf ->
pftri on one GPU, inverse checked through ||A Y - I[:, J]|| on 256 random
columns J with A Y = B (B^H Y) / n + Y.  Prints one JSON line."""
import json, os, sys, time
import numpy as np, torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__))); sys.path.insert(0, ROOT)
from paper_0901_1696_b200 import _capi, convert
n = int(sys.argv[1]) if len(sys.argv) > 1 else 24000
lib = _capi.lib(); dev = torch.device("cuda:0"); st = _capi.stream_handle(dev)
t0 = time.time()
rng = np.random.default_rng(5)
s = np.sqrt(0.5)
bd = torch.empty((n, n), dtype=torch.complex128, device=dev)
rows = 2000
for r0 in range(0, n, rows):  # generate in row slabs to bound host memory
    r1 = min(n, r0 + rows)
    blk = rng.standard_normal((r1 - r0, n)) * s + 1j * (rng.standard_normal((r1 - r0, n)) * s)
    bd[r0:r1].copy_(torch.from_numpy(blk))
gen_s = time.time() - t0
a = bd @ bd.mH
a /= n
a.diagonal().add_(1.0)
r = convert.trttf(a, "L", "C")
del a
info = torch.zeros(1, dtype=torch.int32, device=dev)
torch.cuda.synchronize()
e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
e[0].record()
rc = lib.rfpk_zpftrf(b"C", b"L", n, r.data.data_ptr(), info.data_ptr(), st)
e[1].record()
rc |= lib.rfpk_zpftri(b"C", b"L", n, r.data.data_ptr(), info.data_ptr(), st)
e[2].record()
torch.cuda.synchronize()
assert rc == 0 and int(info.item()) == 0, (rc, int(info.item()))
t_f = e[0].elapsed_time(e[1]); t_i = e[1].elapsed_time(e[2])
# 256 random columns of the inverse from the RFP buffer
J = torch.from_numpy(np.random.default_rng(11).choice(n, 256, replace=False)).to(dev)
full = convert.tfttr(r)                       # lower triangle of A^-1 (column-major)
low = full[:, J]                              # column j: A^-1[j:, j] below the diagonal
up = full[J, :].conj().t()                    # rows j of the lower triangle -> upper part of column j
rowsI = torch.arange(n, device=dev).unsqueeze(1)
Y = torch.where(rowsI >= J.unsqueeze(0), low, up)
del full
AY = bd @ (bd.mH @ Y) / n + Y
E = AY
E[J, torch.arange(256, device=dev)] -= 1.0
err = float(E.abs().max())
fro = float(torch.linalg.norm(E)) / (n * 2.0 ** -53 * 256 ** 0.5)
out = {"config": "c5 complex n=%d 'C' L" % n, "pftrf_ms": t_f, "pftri_ms": t_i,
       "pftrf_tflops": 4 * n ** 3 / 3 / t_f / 1e9, "pftri_tflops": 8 * n ** 3 / 3 / t_i / 1e9,
       "chain_tflops": (4 * n ** 3 / 3 + 8 * n ** 3 / 3) / (t_f + t_i) / 1e9,
       "max_abs_AY_minus_I": err, "fro_scaled_per_col": fro, "gen_s": gen_s}
print(json.dumps(out))
