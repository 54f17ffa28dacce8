import os, sys, torch
sys.path.insert(0, '/root/repo')
from paper_0901_1696_b200 import _capi
lib = _capi.lib(); dev = torch.device("cuda:0"); st = _capi.stream_handle(dev)
info = torch.zeros(1, dtype=torch.int32, device=dev)
bad = 0
for n in (1000, 1500, 2000, 2500, 3000, 4000):
    for seed in range(3):
        torch.manual_seed(n + seed)
        g = torch.randn(n, n, dtype=torch.float64, device=dev)
        a = g @ g.t() / n; a.diagonal().add_(1.0)
        for rep in range(3):
            w = a.clone(); info.zero_()
            rc = lib.rfpk_dpotrf(b"L", w.data_ptr(), n, 1, n, info.data_ptr(), st)
            torch.cuda.synchronize()
            L = torch.tril(w.t())  # column-major lower = row-major upper^T
            err = float((L @ L.t() - a).abs().max())
            if rc or int(info.item()) or err > 1e-10:
                bad += 1
                print("BAD", n, seed, rep, rc, int(info.item()), err, flush=True)
print("bad", bad, "lib", os.environ.get("RFPK_LIB"))
