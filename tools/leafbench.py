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
