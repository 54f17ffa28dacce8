"""Timeline of the tile Cholesky's diagonal chain (developer tool).

  tools/build_variant.sh trace -DRFPK_CHAIN_TRACE
  RFPK_LIB=build/variants/trace.so python tools/chain_trace.py [n ...]

Per diagonal tile d (made by the SUPER task of tile (d, d-1)): %globaltimer
stamps at task start, accumulate done, W_{d-1} flag seen, solve done, leaf
start / end, stores done, done(d, d) published.  Prints the mean of every
interval over the chain's middle tiles."""
import ctypes
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_0901_1696_b200 import _capi  # noqa: E402

lib = _capi.lib()
dev = torch.device("cuda:0")
st = _capi.stream_handle(dev)
info = torch.zeros(1, dtype=torch.int32, device=dev)
CT_EV, CT_MAX = 16, 1024
buf = (ctypes.c_ulonglong * (CT_EV * CT_MAX))()
names = ["start", "acc", "flag", "solve", "leaf0", "leaf1", "stored", "publ"]
for n in [int(x) for x in (sys.argv[1:] or ["2000", "4000"])]:
    torch.manual_seed(n)
    g = torch.randn(n, n, dtype=torch.float64, device=dev)
    a = g @ g.t() / n
    a.diagonal().add_(1.0)
    w = torch.empty_like(a)
    for rep in range(3):
        w.copy_(a)
        lib.rfpk_chain_trace_clear()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        rc = lib.rfpk_dpotrf(b"L", w.data_ptr(), n, 1, n, info.data_ptr(), st)
        e1.record()
        torch.cuda.synchronize()
        assert rc == 0 and int(info.item()) == 0, (rc, int(info.item()))
    ms = e0.elapsed_time(e1)
    lib.rfpk_chain_trace_read(buf, CT_EV * CT_MAX)
    nt = (n + 63) // 64
    t = np.array(buf[: nt * CT_EV], dtype=np.float64).reshape(nt, CT_EV)
    mid = range(max(2, nt // 4), max(3, 3 * nt // 4))
    iv = {"flag wait (publ d-1 -> flag)": [t[d, 2] - t[d - 1, 7] for d in mid],
          "solve (flag -> solve)": [t[d, 3] - t[d, 2] for d in mid],
          "publish+diag update (solve -> leaf0)": [t[d, 4] - t[d, 3] for d in mid],
          "leaf": [t[d, 5] - t[d, 4] for d in mid],
          "stores (leaf1 -> stored)": [t[d, 6] - t[d, 5] for d in mid],
          "publish diag (stored -> publ)": [t[d, 7] - t[d, 6] for d in mid],
          "STEP (publ d-1 -> publ d)": [t[d, 7] - t[d - 1, 7] for d in mid],
          "acc ready before flag (flag - acc)": [t[d, 2] - t[d, 1] for d in mid],
          "  super: start -> acc done (publ d-1 relative)": [t[d, 1] - t[d - 1, 7] for d in mid],
          "  super: acc -> prog ready": [t[d, 13] - t[d, 1] for d in mid],
          "  super: prog -> pready (PARTIAL d)": [t[d, 14] - t[d, 13] for d in mid],
          "  super: pready -> W flag": [t[d, 2] - t[d, 14] for d in mid],
          "  leaf: chol [A11; A21]": [t[d, 8] - t[d, 4] for d in mid],
          "  leaf: A22 -= L21 L21^H": [t[d, 9] - t[d, 8] for d in mid],
          "  leaf: chol32(A22) || inv32(L11), Y": [t[d, 10] - t[d, 9] for d in mid],
          "  leaf: inv32(L22)": [t[d, 11] - t[d, 10] for d in mid],
          "  leaf: W21 = -W22 Y": [t[d, 12] - t[d, 11] for d in mid]}
    print(f"n={n}: {ms:.3f} ms, {nt} diagonal tiles, {ms * 1e3 / nt:.1f} us per tile")
    pub = (t[1:, 7] - t[1, 0]) / 1e3
    print("   diag published at (us from the first SUPER's start), every nt/16 tiles:",
          " ".join(f"{d}:{pub[d - 1]:.0f}" for d in range(1, nt, max(1, nt // 16))))
    for k, v in iv.items():
        print(f"   {np.mean(v) / 1e3:8.2f} us  {k}")
