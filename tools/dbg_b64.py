import sys, numpy as np, torch
sys.path.insert(0, "/root/repo")
from oracle import rfp_oracle as O
from paper_0901_1696_b200 import rfp
n=64
for uplo, tr in [("U","N"),("L","N")]:
    a = O.spd_matrix(n, 1000, "n")
    buf = O.trttf(a, uplo, tr)
    f = buf.copy(); O.pftrf(f, n, uplo, tr)
    arf = torch.from_numpy(np.stack([buf, buf])).cuda()
    info = rfp.pftrf_batched(arf, n, uplo, tr)
    print(uplo, tr, info.tolist())
    g = arf[0].cpu().numpy()
    ds = O.desc(n, uplo, tr)
    for name, x, y in zip(["T1","T2","S1"], O.blocks(g, ds), O.blocks(f, ds)):
        print(name, np.abs(x-y).max())
    # also with the generic kernel path for comparison of T1 only
for uplo, tr in [("U","N"),("L","N"),("U","T"),("L","T")]:
    a = O.spd_matrix(n, 1000, "n")
    buf = O.trttf(a, uplo, tr)
    f = buf.copy(); O.pftrf(f, n, uplo, tr)
    b = np.asfortranarray(np.random.default_rng(0).standard_normal((n, 8)))
    x = b.copy(order="F"); O.pftrs(f, n, uplo, tr, x)
    arf = torch.from_numpy(np.stack([buf, buf])).cuda()
    bt = torch.from_numpy(np.stack([b.T, b.T])).cuda().transpose(1, 2)
    info = rfp.pftrf_pftrs_batched(arf, bt, n, uplo, tr)
    print("fused", uplo, tr, info.tolist(), np.abs(arf[0].cpu().numpy()-f).max(), np.abs(bt[0].cpu().numpy()-x).max())
