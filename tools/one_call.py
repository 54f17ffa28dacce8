"""Run one RFP operation once (for ncu launch lists).
usage: python tools/one_call.py pftrf 16384 L N [d|z] [nrhs]"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_0901_1696_b200 import _capi, convert  # noqa: E402

op, n, uplo, transr = sys.argv[1], int(sys.argv[2]), sys.argv[3], sys.argv[4]
p = sys.argv[5] if len(sys.argv) > 5 else "d"
nrhs = int(sys.argv[6]) if len(sys.argv) > 6 else 64
lib = _capi.lib()
dev = torch.device("cuda:0")
dt = torch.complex128 if p == "z" else torch.float64
g = torch.randn(n, n, dtype=dt, device=dev)
a = g @ g.mH / n
a.diagonal().add_(1.0)
r = convert.trttf(a, uplo, transr)
del a, g
info = torch.zeros(1, dtype=torch.int32, device=dev)
st = _capi.stream_handle(dev)
torch.cuda.synchronize()
if op in ("pftrf", "pftrs", "pftri"):
    getattr(lib, f"rfpk_{p}pftrf")(transr.encode(), uplo.encode(), n, r.data.data_ptr(), info.data_ptr(), st)
if op == "pftrs":
    b = torch.randn(nrhs, n, dtype=dt, device=dev).t()
    torch.cuda.synchronize()
    getattr(lib, f"rfpk_{p}pftrs")(transr.encode(), uplo.encode(), n, nrhs, r.data.data_ptr(), b.data_ptr(), n,
                                   info.data_ptr(), st)
if op == "pftri":
    getattr(lib, f"rfpk_{p}pftri")(transr.encode(), uplo.encode(), n, r.data.data_ptr(), info.data_ptr(), st)
torch.cuda.synchronize()
print("info", int(info.item()))
