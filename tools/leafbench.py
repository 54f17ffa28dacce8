import ctypes, os, torch
lib = ctypes.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "leafbench.so"))
for cplx in (0, 1):
    dt = torch.complex128 if cplx else torch.float64
    g = torch.randn(64, 64, dtype=dt, device="cuda"); a = g @ g.mH + 64 * torch.eye(64, dtype=dt, device="cuda")
    tick = torch.zeros(10, dtype=torch.int64, device="cuda")
    for rep in range(3):
        b = a.clone()
        lib.run_leaf_phases(cplx, ctypes.c_void_p(b.data_ptr()), ctypes.c_void_p(tick.data_ptr()))
    t = tick.cpu().tolist()
    names = ["load", "chol32a", "inv32a", "L21", "herk", "chol32b", "inv32b", "W21", "store"]
    print("cplx" if cplx else "real", " ".join(f"{n}={t[i+1]-t[i]}" for i, n in enumerate(names)), "total", t[-1])
for cplx in (0, 1):
    dt = torch.complex128 if cplx else torch.float64
    g = torch.randn(64, 64, dtype=dt, device="cuda"); a = g @ g.mH + 64 * torch.eye(64, dtype=dt, device="cuda")
    tick = torch.zeros(2, dtype=torch.int64, device="cuda")
    for rep in range(3):
        b = a.clone().t().contiguous().t()  # column-major
        w = torch.zeros(64, 64, dtype=dt, device="cuda")
        lib.run_leaf_full(cplx, ctypes.c_void_p(b.data_ptr()), ctypes.c_void_p(w.data_ptr()), ctypes.c_void_p(tick.data_ptr()))
    L = torch.tril(b); Wm = w.t()  # W stored column-major
    ref = torch.linalg.cholesky(a)
    e1 = float((L - ref).abs().max()); e2 = float((Wm @ L - torch.eye(64, dtype=dt, device="cuda")).abs().max())
    print("full", "cplx" if cplx else "real", "cycles", int(tick[0]), "fail", int(tick[1]), "errL", e1, "errW", e2)
