"""A/B of tuning knobs on one pftrf, or pfsv = pftrf + pftrs(nrhs) when nrhs is
given (default n = 16384 LN): median CUDA-event time on a restored buffer per
knob value, and the largest relative difference to the first value's result.

  python tools/pftrf_ab.py KNOB v1,v2,... [n uplo transr nrhs d|z]"""
import os, sys
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__))); sys.path.insert(0, ROOT)
from paper_0901_1696_b200 import _capi, convert
knob, vals = sys.argv[1], [int(v) for v in sys.argv[2].split(",")]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 16384
uplo = sys.argv[4] if len(sys.argv) > 4 else "L"
transr = sys.argv[5] if len(sys.argv) > 5 else "N"
nrhs = int(sys.argv[6]) if len(sys.argv) > 6 else 0
P = sys.argv[7] if len(sys.argv) > 7 else "d"
DT = torch.complex128 if P == "z" else torch.float64
lib = _capi.lib(); dev = torch.device("cuda:0"); st = _capi.stream_handle(dev)
torch.manual_seed(3)
g = torch.randn(n, n, dtype=DT, device=dev)
a = g @ g.mH / n
a.diagonal().add_(1.0)
r0 = convert.trttf(a, uplo, transr).data
del a, g
r = r0.clone()
b0 = torch.randn(max(nrhs, 1), n, dtype=DT, device=dev).t()
b = b0.clone()
info = torch.zeros(1, dtype=torch.int32, device=dev)
ref = None
for v in vals:
    _capi.set_tuning(knob, v)
    ts = []
    for rep in range(int(os.environ.get('REPS', '6'))):
        r.copy_(r0)
        b.copy_(b0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        if nrhs:
            rc = getattr(lib, f"rfpk_{P}pfsv")(transr.encode(), uplo.encode(), n, nrhs, r.data_ptr(), b.data_ptr(),
                                n, info.data_ptr(), st)
        else:
            rc = getattr(lib, f"rfpk_{P}pftrf")(transr.encode(), uplo.encode(), n, r.data_ptr(), info.data_ptr(), st)
        e1.record()
        torch.cuda.synchronize()
        assert rc == 0 and int(info.item()) == 0
        ts.append(e0.elapsed_time(e1))
    out = b if nrhs else r
    if ref is None:
        ref = out.clone()
    d = float((out - ref).abs().max() / ref.abs().max())
    print(f"{knob} = {v}: {'pfsv' if nrhs else 'pftrf'} {sorted(ts)[len(ts) // 2]:.3f} ms (min {min(ts):.3f}), "
          f"max rel diff vs first {d:.1e}")
