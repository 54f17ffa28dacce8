#!/usr/bin/env python
"""Benchmark contract for the B200 RFPF path.

Headline = BASELINE config 3 (the north-star target): one real FP64 SPD
matrix, n = 16384, TRANSR='N', UPLO='L', A = B Bᵀ/n + I; a step is pftrf
followed by pftrs with nrhs = 1024 (ONE C-ABI call, rfpk_dpfsv) on an RFP
buffer restored from a pristine device copy at the start of the step (the
1.07 GB RFP buffer and the RHS exceed the 126 MB L2: no flush needed).
Metric: FP64 GFLOP/s, LAPACK flop model n³/3 + 2n²·nrhs.

The same JSON line carries
* ``roofline``: the DOMINANT kernel of the step (most device time in the
  library's kernel clock, tile_trsm_kernel) over all its launches, timed live
  on the streams they run on, against the nominal FP64 peak; ``kernels``
  lists every kernel of the step the same way and ``phases`` the SRPA steps;
* ``batched``: config 4 (65,536 x n = 64 UN, pftrf + pftrs(8)) sharded by
  matrix over the N ranks, with the NCCL gather of per-matrix info and
  residual timed separately;
* ``per_config`` (N = 1): configs 1, 2 (8 layouts), 5 and the conversions;
* ``cpu_baseline`` (N = 1): the unmodified reference (baseline/_ref), one
  full-size config-3 rep through its public ``rfp.pftrf`` / ``rfp.pftrs``.

  python bench.py [--gpus N --steps K --warmup W] [--impl reference]

Under torchrun (N > 1) every rank factors its own config-3 replica (single
matrices do not shard: "replicas only", weak scaling) and config 4 is split
by matrix.  ``--impl reference`` times the reference's own CPU path on the
host cores: each step is ONE call of the reference's 10-call SRPA composition
of config 3 at FULL size (rfp.py:70-89 then :118-136, through the
reference's own ``kernels`` on its ``_views``), cycling through the
composition, so K = 10 steps make one whole pftrf + pftrs.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

NOMINAL_FP64_TFLOPS = 37.2  # 148 SM x 128 flop/clk x 1.965 GHz (B200_PROFILING / SURVEY 6)
METRIC = "FP64 GFLOP/s of RFPF pftrf+pftrs (n=16384, TRANSR=N, UPLO=L, nrhs=1024)"
C3_N, C3_NRHS = 16384, 1024


def load_json(name):
    try:
        with open(os.path.join(ROOT, *name.split("/"))) as f:
            return json.load(f)
    except Exception:
        return {}


def hbm_peak():
    return float(load_json("MEASURED_PEAKS.json").get("hbm_gbs", 6553.9))


def ncu_bytes(label):
    """DRAM bytes (read + write) per launch of the kernel with this kernel-
    clock label, from the committed ncu capture (profiles/ncu_traffic.json),
    or None."""
    e = load_json("profiles/ncu_traffic.json").get(label)
    return e.get("bytes") if isinstance(e, dict) else None


# ---------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi sampling during the timed region (B200_PROFILING recipe)."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            t0 = time.time()
            while not self.lines and time.time() - t0 < 2.0:  # first sample before timing
                time.sleep(0.02)
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            n0 = len(self.lines)
            t0 = time.time()
            while len(self.lines) <= n0 and time.time() - t0 < 1.0:  # one sample after
                time.sleep(0.02)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            p = [x.strip() for x in ln.split(",")]
            if len(p) < 7:
                continue
            try:
                sm.append(float(p[0]))
                mx.append(float(p[1]))
            except ValueError:
                continue
            for nm, v in zip(names, p[3:7]):
                if v.lower() in ("active", "1"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": float(max(mx)),
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------- dist
def _backend():
    """NCCL on the GPUs; BENCH_DIST_BACKEND=gloo lets the CPU tests drive the
    rank logic (barrier, max over ranks, gathers) with world_size 2."""
    return os.environ.get("BENCH_DIST_BACKEND", "nccl")


def _coll_device():
    return "cuda" if _backend() == "nccl" else "cpu"


def dist_env():
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def dist_setup():
    rank, world, local = dist_env()
    if world > 1:
        import torch
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if _backend() == "nccl":
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(_backend())
    return rank, world, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(x, world):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device=_coll_device())
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def all_ranks(x, world):
    if world == 1:
        return [x]
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device=_coll_device())
    out = [torch.zeros_like(t) for _ in range(world)]
    dist.all_gather(out, t)
    return [float(v.item()) for v in out]


# ---------------------------------------------------------------- CPU reference
REF_DIR = os.path.join(ROOT, "baseline", "_ref")


def _reference_module():
    """The UNMODIFIED reference package installed by `pip install --target
    baseline/_ref /root/reference/pkg` (git-ignored; travels with gpurun), or
    None when absent."""
    if not os.path.isdir(os.path.join(REF_DIR, "rfpk")):
        return None
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    try:
        import rfpk.convert
        import rfpk.kernels
        import rfpk.rfp
        return rfpk
    except Exception:
        return None


def _threads():
    try:
        from threadpoolctl import threadpool_info
        return max([d.get("num_threads", 1) for d in threadpool_info()] + [1])
    except Exception:
        return os.cpu_count()


def _host_c3(n, nrhs, seed=3):
    """Config 3's A (B Bᵀ/n + I, B ~ N(0,1) seeded; one host SYRK, the lower
    triangle is what trttf 'L' reads) and its right-hand side."""
    from scipy.linalg.blas import dsyrk
    rng = np.random.default_rng(seed)
    b = rng.standard_normal((n, n))
    a = np.asfortranarray(dsyrk(1.0, b, lower=1))
    del b
    a /= n
    a[np.diag_indices(n)] += 1.0
    x = np.asfortranarray(rng.standard_normal((n, nrhs)))
    return a, x


def c3_calls(ref, r, x):
    """The reference's pftrf + pftrs composition for UPLO='L' as its 10
    kernel calls on its own views (rfp.py:70-89, :118-136), with the
    LAPACK-model flops of each."""
    K = ref.kernels
    t1, t2, s1 = ref.rfp._views(r)
    n1, n2, m = r.desc.n1, r.desc.n2, x.shape[1]
    b1, b2 = x[:n1], x[n1:]
    return [
        ("potrf(T1)", n1 ** 3 / 3, lambda: K.potrf_ref("L", t1)),
        ("trsm(S1)", n1 * n1 * n2, lambda: K.trsm("R", "L", "C", "N", 1.0, t1, s1)),
        ("syrk(T2)", n2 * n2 * n1, lambda: K.syrk_herk("U", "C", -1.0, s1.T, 1.0, t2, hermitian=False)),
        ("potrf(T2)", n2 ** 3 / 3, lambda: K.potrf_ref("U", t2)),
        ("trsm1", n1 * n1 * m, lambda: K.trsm("L", "L", "N", "N", 1.0, t1, b1)),
        ("gemm1", 2 * n2 * n1 * m, lambda: K.gemm("N", "N", -1.0, s1, b1, 1.0, b2)),
        ("trsm2", n2 * n2 * m, lambda: K.trsm("L", "U", "T", "N", 1.0, t2, b2)),
        ("trsm3", n2 * n2 * m, lambda: K.trsm("L", "L", "C", "N", 1.0, t2.T, b2)),
        ("gemm2", 2 * n1 * n2 * m, lambda: K.gemm("C", "N", -1.0, s1, b2, 1.0, b1)),
        ("trsm4", n1 * n1 * m, lambda: K.trsm("L", "L", "C", "N", 1.0, t1, b1)),
    ]


def cpu_baseline_c3(n=C3_N, nrhs=C3_NRHS):
    """One full-size config-3 rep of the unmodified reference through its
    public API (rfp.pftrf then rfp.pftrs), timed around the two calls only
    (SPEC.md:412).  Falls back to the oracle port when baseline/_ref is
    absent."""
    ref = _reference_module()
    a, x = _host_c3(n, nrhs)
    if ref is not None:
        r = ref.convert.trttf(a, "L", "N")
        del a
        t0 = time.perf_counter()
        assert ref.rfp.pftrf(r) == 0
        t1 = time.perf_counter()
        ref.rfp.pftrs(r, x)
        t2 = time.perf_counter()
    else:
        from oracle import rfp_oracle as O
        buf = O.trttf(a, "L", "N")
        del a
        t0 = time.perf_counter()
        assert O.pftrf(buf, n, "L", "N") == 0
        t1 = time.perf_counter()
        O.pftrs(buf, n, "L", "N", x)
        t2 = time.perf_counter()
    flops = n ** 3 / 3 + 2 * n * n * nrhs
    cores = _threads()
    who = "reference rfpk (baseline/_ref) public rfp.pftrf + rfp.pftrs" if ref is not None \
        else "oracle port pftrf + pftrs"
    return {"value": flops / (t2 - t0) / 1e9, "unit": "GFLOP/s", "cores": cores,
            "kind": "reference" if ref is not None else "port",
            "sample": f"{who}, ONE full-size rep of config 3 (n={n}, nrhs={nrhs}): pftrf "
                      f"{t1 - t0:.1f} s + pftrs {t2 - t1:.1f} s; numpy/OpenBLAS {cores} threads, "
                      f"{os.cpu_count()} host CPUs"}


def run_reference(args, rank, world):
    """--impl reference: rank 0 times the reference's own CPU path on config 3
    at full size, one SRPA call per step (see the module docstring)."""
    if rank != 0:
        return
    ref = _reference_module()
    if ref is None:
        print(json.dumps({"impl": "reference", "unavailable":
                          "baseline/_ref missing (pip install --target baseline/_ref /root/reference/pkg)"}))
        return
    # warm-up: whole compositions at a small order (imports, thread pools)
    for _ in range(args.warmup):
        aw, xw = _host_c3(1024, 64, seed=5)
        rw = ref.convert.trttf(aw, "L", "N")
        for _, _, f in c3_calls(ref, rw, xw):
            f()
    a, x0 = _host_c3(C3_N, C3_NRHS)
    r = ref.convert.trttf(a, "L", "N")
    del a
    pristine = r.data.copy()
    x = x0.copy(order="F")
    calls = c3_calls(ref, r, x)
    flops, secs, done = 0.0, 0.0, []
    for i in range(args.steps):
        k = i % len(calls)
        if k == 0 and i:
            r.data[:] = pristine          # restore (outside the timed call)
            x[:] = x0
        name, fl, f = calls[k]
        t0 = time.perf_counter()
        f()
        dt = time.perf_counter() - t0
        flops += fl
        secs += dt
        done.append(name)
    value = flops / secs / 1e9
    cores = _threads()
    rem = args.steps % len(calls)
    sample = (f"{args.steps} steps = {args.steps / len(calls):.1f} passes over the reference's "
              f"10-call config-3 composition at FULL size (n={C3_N}, nrhs={C3_NRHS}), one call per "
              f"step ({'whole passes' if rem == 0 else 'last pass partial: ' + ','.join(done[-rem:])}); "
              f"numpy/OpenBLAS {cores} threads, {os.cpu_count()} host CPUs")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "GFLOP/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": secs / args.steps * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded numpy, host-built A)",
        "config": c3_config(world),
        "cpu_baseline": {"value": value, "unit": "GFLOP/s", "cores": cores, "kind": "reference",
                         "sample": sample},
        "e2e": {"value": value, "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def c3_config(world):
    return {"workload": "BASELINE config 3: pftrf+pftrs, n=16384, TRANSR=N, UPLO=L, nrhs=1024",
            "n": C3_N, "nrhs": C3_NRHS, "transr": "N", "uplo": "L",
            "l2": "no flush: RFP buffer 1.07 GB + RHS 134 MB exceed the 126 MB L2",
            "call": "rfpk_dpfsv (pftrf + pftrs in one C-ABI call; e2e: rfpk_dpfsv_host)",
            "parallelism": f"replicas x{world}" if world > 1 else "single GPU"}


# ---------------------------------------------------------------- GPU helpers
def ev_time(fn, reps, setup=None):
    """Median CUDA-event time (ms) of fn() on the current stream over `reps`
    runs after one warm-up; `setup` (untimed) runs before each."""
    import torch
    ts = []
    for i in range(reps + 1):
        if setup:
            setup()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        e.synchronize()
        if i:
            ts.append(s.elapsed_time(e))
    return float(np.median(ts))


def kernel_flops(name, dims):
    """LAPACK-model flops of one library kernel launch from its kernel-clock
    label (None: a data-movement kernel)."""
    d = [int(v) for v in dims.split("x")]
    if name == "tile_trsm":
        return d[0] * d[0] * d[1]
    if name == "tile_potrf":           # m x ncols panel: ncols³/3 + (m - ncols)·ncols²
        m, c = d
        return c ** 3 / 3 + (m - c) * c * c
    if name == "syrk":
        return d[0] * d[1] * d[2]      # one triangle of an M x N output, rank K
    if name in ("gemm", "gemm_splitk"):
        return 2 * d[0] * d[1] * d[2]
    return None


def kernel_table(table, steps):
    """Per-kernel rows (name, shape, launches per step, ms per step, TFLOP/s)
    from the phase clock's "kernel ..." labels, heaviest first."""
    rows = []
    for lab, (ms, cnt) in table.items():
        if not lab.startswith("kernel "):
            continue
        _, name, dims = lab.split(" ")
        fl = kernel_flops(name, dims)
        row = {"kernel": name, "shape": dims, "launches_per_step": cnt / steps,
               "ms_per_step": ms / steps, "ms_per_launch": ms / cnt}
        if fl is not None:
            row["tflops"] = fl * cnt / (ms * 1e-3) / 1e12
            row["frac_nominal"] = row["tflops"] / NOMINAL_FP64_TFLOPS
            row["flops_per_launch"] = fl
        b = ncu_bytes(lab)
        if b is not None:
            row["dram_bytes_per_launch"] = b
        rows.append(row)
    rows.sort(key=lambda r: -r["ms_per_step"])
    return rows


C3_PHASE_FLOPS = {
    # SRPA steps of config 3 (n1 = n2 = 8192, nrhs = 1024) -> LAPACK-model flops
    "pftrf potrf(T1)||trsm(S1)": lambda n1, n2, m: n1 ** 3 / 3 + n1 * n1 * n2,
    "pftrf syrk(T2)": lambda n1, n2, m: n2 * n2 * n1,
    "pftrf potrf(T2)||pftrs(T1,S1)": lambda n1, n2, m: n2 ** 3 / 3 + n1 * n1 * m + 2 * n1 * n2 * m,
    "pftrs trsm2": lambda n1, n2, m: n2 * n2 * m,
    "pftrs trsm3": lambda n1, n2, m: n2 * n2 * m,
    "pftrs gemm2": lambda n1, n2, m: 2 * n1 * n2 * m,
    "pftrs trsm4": lambda n1, n2, m: n1 * n1 * m,
}


def phase_table(table, steps, n1, n2, m, dgemm):
    rows = []
    for lab, (ms, cnt) in table.items():
        if lab.startswith("kernel "):
            continue
        row = {"phase": lab, "ms_per_step": ms / steps}
        f = C3_PHASE_FLOPS.get(lab)
        if f:
            fl = f(n1, n2, m)
            row["flops"] = fl
            row["tflops"] = fl * cnt / (ms * 1e-3) / 1e12
            row["frac_nominal"] = row["tflops"] / NOMINAL_FP64_TFLOPS
            row["frac_measured_dgemm"] = row["tflops"] / dgemm
        rows.append(row)
    rows.sort(key=lambda r: -r["ms_per_step"])
    return rows


def measured_dgemm(dev):
    """cuBLAS DGEMM 8192³ through torch (the measured FP64 ceiling, context)."""
    import torch
    g1 = torch.randn(8192, 8192, dtype=torch.float64, device=dev)
    g2 = torch.randn(8192, 8192, dtype=torch.float64, device=dev)
    ms = ev_time(lambda: torch.matmul(g1, g2), 3)
    return 2 * 8192 ** 3 / (ms * 1e-3) / 1e12


# ---------------------------------------------------------------- config 3 (headline)
def run_c3(args, rank, world, local):
    import torch
    from paper_0901_1696_b200 import _capi, convert, rfp

    lib = _capi.lib()
    dev = torch.device("cuda", local)
    n, nrhs, uplo, transr = C3_N, C3_NRHS, "L", "N"
    n1, n2 = (n + 1) // 2, n // 2
    flops = n ** 3 / 3 + 2 * n * n * nrhs

    # inputs: B ~ N(0,1) seeded on the host, A = B Bᵀ/n + I formed on the device
    seed = 1234 + rank
    bd = torch.from_numpy(np.random.default_rng(seed).standard_normal((n, n))).to(dev)
    a = bd @ bd.t()
    del bd
    a /= n
    a.diagonal().add_(1.0)
    pristine = convert.trttf(a, uplo, transr).data  # our trttf kernel
    rhs0 = torch.from_numpy(np.random.default_rng(seed + 7).standard_normal((nrhs, n))).to(dev).t()
    work = torch.empty_like(pristine)
    x = torch.empty((nrhs, n), dtype=torch.float64, device=dev).t()
    info = torch.zeros(1, dtype=torch.int32, device=dev)
    st = torch.cuda.current_stream(dev)
    sh = st.cuda_stream
    T, U = transr.encode(), uplo.encode()

    def step():
        work.copy_(pristine)
        x.copy_(rhs0)
        rc = lib.rfpk_dpfsv(T, U, n, nrhs, work.data_ptr(), x.data_ptr(), n, info.data_ptr(), sh)
        if rc:
            raise RuntimeError(f"rfpk_dpfsv failed rc={rc}")

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    assert int(info.item()) == 0, "factorization failed"

    barrier(world)
    torch.cuda.synchronize()
    l0 = lib.rfpk_launch_count()
    # kernel clock: event pairs around every library launch, on its stream,
    # read after the loop (no synchronisation inside the timed region)
    with _capi.phase_clock() as pc:
        with ClockSampler(local) as clk:
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record(st)
            for _ in range(args.steps):
                step()
            e.record(st)
            torch.cuda.synchronize()
    launches = lib.rfpk_launch_count() - l0
    table = pc.table()
    barrier(world)
    ms = max_over_ranks(s.elapsed_time(e) / args.steps, world)
    value = world * flops / (ms * 1e-3) / 1e9

    # result check: ||A X - B|| / (||A|| ||X|| n eps) on the last step's solution
    resid = float((a @ x - rhs0).norm() / (a.norm() * x.norm() * n * 2.0 ** -53))
    del a
    dgemm = measured_dgemm(dev)

    # the dominant kernel's largest launch ALONE (pftrf's S1 solve, n2 x n1
    # right-hand sides on the factored T1 of the last step's buffer, as pftrf
    # issues it): the in-step launch below shares the SMs with potrf(T1)
    ld = n + 1 - (n & 1)
    shift = 1 - (n & 1)
    t1p = work.data_ptr() + 8 * shift
    s1p = work.data_ptr() + 8 * (n1 + shift)

    def s1_solve():
        rc = lib.rfpk_dtrsm(b"R", b"L", b"C", b"N", 1.0, t1p, n1, 1, ld, s1p, n2, n1, 1, ld,
                            info.data_ptr(), sh)
        if rc:
            raise RuntimeError(f"rfpk_dtrsm failed rc={rc}")

    alone_ms = ev_time(s1_solve, 3)
    alone_tf = n1 * n1 * n2 / (alone_ms * 1e-3) / 1e12

    kernels = kernel_table(table, args.steps)
    phases = phase_table(table, args.steps, n1, n2, nrhs, dgemm)
    # the dominant kernel: the most device time per step summed over its
    # launches (tile_trsm_kernel: the S1 solve beside potrf(T1) and pftrs's
    # four solves)
    by_name = {}
    for r_ in kernels:
        by_name.setdefault(r_["kernel"], []).append(r_)
    dom = max(by_name, key=lambda k: sum(r_["ms_per_step"] for r_ in by_name[k]))
    drows = by_name[dom]
    d_ms = sum(r_["ms_per_step"] for r_ in drows)
    d_fl = sum(r_.get("flops_per_launch", 0) * r_["launches_per_step"] for r_ in drows)
    d_launches = sum(r_["launches_per_step"] for r_ in drows)
    d_bytes = [r_.get("dram_bytes_per_launch") for r_ in drows]
    traffic = (sum(b * r_["launches_per_step"] for b, r_ in zip(d_bytes, drows)) / d_launches
               if all(b is not None for b in d_bytes) else None)
    achieved = d_fl / (d_ms * 1e-3) / 1e12
    roofline = {
        "bound": "tensor", "kernel": f"{dom}_kernel (all {d_launches:g} launches per step)",
        "achieved": achieved, "peak": NOMINAL_FP64_TFLOPS, "unit": "TFLOP/s",
        "frac": achieved / NOMINAL_FP64_TFLOPS, "traffic": traffic,
        "algorithmic_flops_per_launch": d_fl / d_launches, "ms_per_launch": d_ms / d_launches,
        "launches": [{k: r_[k] for k in ("shape", "launches_per_step", "ms_per_launch", "tflops",
                                         "frac_nominal") if k in r_} for r_ in drows],
        "alone": {"launch": f"S1 solve {n2}x{n1} by itself (rfpk_dtrsm on the same views, median "
                            "of 3 after the timed steps)", "ms_per_launch": alone_ms,
                  "achieved": alone_tf, "frac": alone_tf / NOMINAL_FP64_TFLOPS,
                  "frac_measured_dgemm": alone_tf / dgemm},
        "timing": ("live: CUDA events around every launch on the stream it runs on, inside the "
                   f"{args.steps} timed steps (the S1 solve's launch spans its run beside "
                   "potrf(T1), flag waits included)"),
        "peak_source": "nominal FP64 DMMA 148 SM x 128 flop/clk x 1.965 GHz (MEASURED_PEAKS.json "
                       f"has no FP64 figure); measured cuBLAS DGEMM here: {dgemm:.2f} TFLOP/s",
        "traffic_source": "ncu dram__bytes_read.sum + dram__bytes_write.sum per launch, launch-"
                          "weighted (profiles/ncu_traffic.json)",
    }

    line = {
        "metric": METRIC, "value": value, "unit": "GFLOP/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic: B~N(0,1) seeded numpy, A=B B^T/n+I (formed on device), RHS~N(0,1)",
        "config": c3_config(world),
        "fraction_of_fp64_nominal": value / world / 1e3 / NOMINAL_FP64_TFLOPS,
        "fraction_of_fp64_measured_dgemm": value / world / 1e3 / dgemm,
        "roofline": roofline,
        "kernels": kernels,
        "phases": phases,
        "residual_scaled": resid,
        "gpu_launches": launches,
        "clocks": clk.summary(),
    }
    if args.no_e2e:  # (profiling runs: kernels gated on copy-engine flags)
        return line
    # end-to-end through the public Python API with host (pinned) buffers
    host_rfp = pristine.cpu().pin_memory()
    host_b = rhs0.t().contiguous().cpu().pin_memory()  # nrhs x n row-major == column-major B
    h2d = host_rfp.numel() * 8 + host_b.numel() * 8
    d2h = host_b.numel() * 8
    out_x = torch.empty_like(host_b).pin_memory()
    e2e_steps = max(1, args.steps // 2)

    def e2e_step():
        # one public call: pftrf + pftrs from pinned host memory, every copy
        # overlapped with the computation by the library (rfp.pfsv_from_host)
        _, inf = rfp.pfsv_from_host(host_rfp, host_b.t(), n, uplo, transr, out=out_x.t())
        assert inf == 0

    e2e_step()
    barrier(world)
    torch.cuda.synchronize()
    es, ee = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    es.record(st)
    for _ in range(e2e_steps):
        e2e_step()
    ee.record(st)
    torch.cuda.synchronize()
    e2e_ms = max_over_ranks(es.elapsed_time(ee) / e2e_steps, world)
    # the host path's solution against the device step's (same kernels, same
    # summation order: expected bit-identical; the head block came back row
    # block by row block while the last solve still ran)
    xd = x.t().contiguous().cpu()
    e2e_diff = float((out_x - xd).abs().max() / xd.abs().max())
    del pristine, work, host_rfp
    line["e2e"] = {"value": world * flops / (e2e_ms * 1e-3) / 1e9, "unit": "GFLOP/s",
                   "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "ms_per_step": e2e_ms,
                   "max_rel_diff_vs_device_solution": e2e_diff,
                   "path": "rfp.pfsv_from_host (public API): pinned host RFP + RHS in, solution "
                           "out, transfers overlapped with pftrf/pftrs"}
    return line


# ---------------------------------------------------------------- config 4 (sharded batch)
def make_c4_inputs(start, stop, n, nrhs, seed0, dev):
    """A_k = B_k B_kᵀ + n I with B_k ~ N(0,1) from default_rng(seed0 + k)
    (BASELINE config 4; the right-hand side follows from the same
    generator); returns (full A (count, n, n), RFP (count, nt), B (count, n,
    nrhs) with unit stride along n)."""
    import torch
    from paper_0901_1696_b200.layout import make_descriptor, map_index
    count = stop - start
    bh = np.empty((count, n, n))
    rh = np.empty((count, nrhs, n))
    for k in range(count):
        g = np.random.default_rng(seed0 + start + k)
        bh[k] = g.standard_normal((n, n))
        rh[k] = g.standard_normal((nrhs, n))
    bd = torch.from_numpy(bh).to(dev)
    a = torch.bmm(bd, bd.transpose(1, 2))
    a.diagonal(dim1=1, dim2=2).add_(float(n))
    del bd
    d = make_descriptor(n, "U", "N")
    idx = np.empty(d.nt, dtype=np.int64)  # RFP slot -> column-major offset (product layout map)
    for j in range(1, n + 1):
        for i in range(1, j + 1):
            idx[map_index(d, i, j) - 1] = (i - 1) + (j - 1) * n
    arf = a.transpose(1, 2).reshape(count, n * n)[:, torch.from_numpy(idx).to(dev)].contiguous()
    rhs = torch.from_numpy(rh).to(dev).transpose(1, 2)
    return a, arf, rhs


def cpu_baseline_c4(arf_host, rhs_host, n, nrhs, sample=2048):
    """Config 4 on the host: the unmodified reference's rfp.pftrf + rfp.pftrs
    per matrix (rfp.py:55-136) over the first `sample` matrices of the same
    inputs, ONE process (the reference has no batched entry point; a matrix of
    order 64 is interpreter-bound, so its BLAS threads do not help)."""
    ref = _reference_module()
    m = min(sample, arf_host.shape[0])
    t0 = time.perf_counter()
    if ref is not None:
        desc = ref.layout.make_descriptor(n, "U", "N")
        for k in range(m):
            r = ref.convert.RfpTriangle(arf_host[k].copy(), desc)
            assert ref.rfp.pftrf(r) == 0
            ref.rfp.pftrs(r, np.asfortranarray(rhs_host[k]))
    else:
        from oracle import rfp_oracle as O
        for k in range(m):
            buf = arf_host[k].copy()
            assert O.pftrf(buf, n, "U", "N") == 0
            O.pftrs(buf, n, "U", "N", np.asfortranarray(rhs_host[k]))
    dt = time.perf_counter() - t0
    return {"value": m / dt, "unit": "matrices/s", "cores": 1,
            "kind": "reference" if ref is not None else "port",
            "sample": f"first {m} of the 65,536 matrices, one host process, "
                      f"{'reference rfpk (baseline/_ref)' if ref is not None else 'oracle port'} "
                      f"rfp.pftrf + rfp.pftrs(nrhs={nrhs}) per matrix: {dt:.2f} s"}


def run_c4(args, rank, world, local):
    """Config 4: 65,536 independent n = 64 matrices sharded by contiguous
    ranges; one fused batched launch per step per rank; the only collective
    is the NCCL all-gather of per-matrix (info, residual) after the timed
    region, timed on the device."""
    import torch
    from paper_0901_1696_b200 import _capi, rfp
    from paper_0901_1696_b200.shard import gather_results, shard_range

    lib = _capi.lib()
    dev = torch.device("cuda", local)
    total, n, nrhs = args.batch, 64, 8
    start, stop = shard_range(total, rank, world)
    count = stop - start
    nt = n * (n + 1) // 2
    a, arf0, rhs0 = make_c4_inputs(start, stop, n, nrhs, 20260000, dev)
    steps = args.steps
    # every timed step factors its own fresh copy (no restore inside the
    # timed region; 1.36 GB per step at N = 1 keeps each step out of L2)
    nbuf = 2 + steps
    arfs = [arf0.clone() for _ in range(nbuf)]
    rhss = [rhs0.clone() for _ in range(nbuf)]
    info = torch.zeros(count, dtype=torch.int32, device=dev)
    st = torch.cuda.current_stream(dev)
    sh = st.cuda_stream

    def step(i):
        rc = lib.rfpk_dpftrf_pftrs_batched(b"N", b"U", n, nrhs, arfs[i].data_ptr(), nt,
                                           rhss[i].data_ptr(), n, n * nrhs, count,
                                           info.data_ptr(), sh)
        if rc:
            raise RuntimeError(f"rfpk_dpftrf_pftrs_batched rc={rc}")

    for i in range(2):
        step(i)
    torch.cuda.synchronize()
    barrier(world)
    torch.cuda.synchronize()
    l0 = lib.rfpk_launch_count()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(st)
    for i in range(2, nbuf):
        step(i)
    e.record(st)
    torch.cuda.synchronize()
    launches = lib.rfpk_launch_count() - l0
    my_ms = s.elapsed_time(e) / steps
    per_rank_ms = all_ranks(my_ms, world)
    ms = max(per_rank_ms)

    # per-matrix scaled residual ||A x - b||_max / (||A||_max ||x||_max n eps)
    x = rhss[-1]
    r = torch.bmm(a, x) - rhs0
    resid = r.abs().amax(dim=(1, 2)) / (a.abs().amax(dim=(1, 2)) * x.abs().amax(dim=(1, 2)) * n * 2.0 ** -53)
    del arfs, rhss, a
    torch.cuda.synchronize()
    barrier(world)
    gs, ge = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    gs.record(st)
    gi, gr = gather_results(info, resid, total) if world > 1 else (info, resid)
    ge.record(st)
    torch.cuda.synchronize()
    gather_ms = max_over_ranks(gs.elapsed_time(ge), world)

    per_matrix_bytes = 2 * nt * 8 + 2 * n * nrhs * 8
    # HBM fraction of the slowest rank's kernel (its own shard's bytes)
    shard_max = -(-total // world)
    gbs = shard_max * per_matrix_bytes / (ms * 1e-3) / 1e9
    block = {
        "workload": "BASELINE config 4: 65536 x n=64 UN pftrf+pftrs(nrhs=8), contiguous shards, "
                    "NCCL all_gather_into_tensor of (info, residual) after compute",
        "matrices": total, "n_ranks": world, "value": total / (ms * 1e-3), "unit": "matrices/s",
        "ms_per_step": ms, "per_rank_ms": per_rank_ms, "steps": steps,
        "gather_ms": gather_ms, "gather_bytes": total * 16,
        "roofline": {"bound": "hbm", "kernel": "batched64_kernel (fused pftrf+pftrs)",
                     "achieved": gbs, "peak": hbm_peak(), "unit": "GB/s", "frac": gbs / hbm_peak(),
                     "bytes_per_matrix": per_matrix_bytes,
                     "traffic": ncu_bytes("kernel batched64 65536x8") if count == 65536 else None},
        "gpu_launches": launches,
        "data": "synthetic: B_k~N(0,1) from default_rng(20260000+k), A_k=B_k B_k^T+64 I",
    }
    if rank == 0:
        block["failed_matrices"] = int((gi != 0).sum())
        block["max_residual_scaled"] = float(gr.max())
    if rank == 0 and world == 1 and not args.no_cpu:
        m = min(2048, count)
        block["cpu_baseline"] = cpu_baseline_c4(arf0[:m].cpu().numpy(), rhs0[:m].cpu().numpy(),
                                                n, nrhs, m)
    if args.no_e2e:
        return block
    # e2e through the public API with pinned host buffers
    host_arf = arf0.cpu().pin_memory()
    host_b = rhs0.transpose(1, 2).contiguous().cpu().pin_memory()  # (count, nrhs, n)
    out_b = torch.empty_like(host_b).pin_memory()

    def e2e_step():
        _, inf = rfp.pftrf_pftrs_batched_from_host(host_arf, "N", "U", n, host_b.transpose(1, 2),
                                                   out=out_b.transpose(1, 2))
        torch.cuda.current_stream().synchronize()
        return inf

    e2e_step()
    barrier(world)
    es, ee = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e2e_steps = max(1, steps // 2)
    es.record(st)
    for _ in range(e2e_steps):
        e2e_step()
    ee.record(st)
    torch.cuda.synchronize()
    e2e_ms = max_over_ranks(es.elapsed_time(ee) / e2e_steps, world)
    block["e2e"] = {"value": total / (e2e_ms * 1e-3), "unit": "matrices/s",
                    "h2d_bytes_per_step": host_arf.numel() * 8 + host_b.numel() * 8,
                    "d2h_bytes_per_step": host_b.numel() * 8, "ms_per_step": e2e_ms,
                    "path": "rfp.pftrf_pftrs_batched_from_host (chunked, copies overlapped)"}
    return block


# ---------------------------------------------------------------- per-config blocks (N = 1)
def per_config(dev):
    import torch
    from paper_0901_1696_b200 import _capi, convert

    lib = _capi.lib()
    sh = lambda: torch.cuda.current_stream(dev).cuda_stream  # noqa: E731
    info = torch.zeros(1, dtype=torch.int32, device=dev)
    out = {}

    def spd(n, scale, cplx=False, seed=0):
        g = torch.Generator(device=dev).manual_seed(seed)
        if cplx:
            b = torch.complex(torch.randn(n, n, dtype=torch.float64, device=dev, generator=g),
                              torch.randn(n, n, dtype=torch.float64, device=dev, generator=g))
            b *= 0.5 ** 0.5
        else:
            b = torch.randn(n, n, dtype=torch.float64, device=dev, generator=g)
        a = b @ b.mH
        del b
        if scale == "n":
            a.diagonal().add_(float(n))
        else:
            a /= n
            a.diagonal().add_(1.0)
        return a

    def rfp_ops(n, uplo, transr, nrhs, pftri, reps=10):
        a = spd(n, "n", False, seed=n)
        r = convert.trttf(a, uplo, transr)
        del a
        pristine = r.data.clone()
        T, U = transr.encode(), uplo.encode()
        res = {}
        ms = ev_time(lambda: lib.rfpk_dpftrf(T, U, n, r.data.data_ptr(), info.data_ptr(), sh()),
                     reps, lambda: r.data.copy_(pristine))
        assert int(info.item()) == 0
        res["pftrf_ms"] = ms
        res["pftrf_tflops"] = n ** 3 / 3 / ms / 1e9
        fac = r.data.clone()
        if nrhs:
            b0 = torch.randn(nrhs, n, dtype=torch.float64, device=dev).t()
            b = b0.clone()
            ms = ev_time(lambda: lib.rfpk_dpftrs(T, U, n, nrhs, r.data.data_ptr(), b.data_ptr(), n,
                                                 info.data_ptr(), sh()), reps, lambda: b.copy_(b0))
            res["pftrs_ms"] = ms
            res["pftrs_tflops"] = 2 * n * n * nrhs / ms / 1e9
            res["nrhs"] = nrhs
        if pftri:
            ms = ev_time(lambda: lib.rfpk_dpftri(T, U, n, r.data.data_ptr(), info.data_ptr(), sh()),
                         reps, lambda: r.data.copy_(fac))
            assert int(info.item()) == 0
            res["pftri_ms"] = ms
            res["pftri_tflops"] = 2 * n ** 3 / 3 / ms / 1e9
        return res

    # config 1
    c1 = rfp_ops(1000, "L", "N", 100, True, reps=20)
    c1["workload"] = "config 1: n=1000 LN pftrf, pftrs(100), pftri (median of 20, graph replays)"
    out["c1"] = c1
    # config 2: the 8 variants
    rows = []
    for n in (4000, 4001):
        for uplo in "LU":
            for transr in "NT":
                res = rfp_ops(n, uplo, transr, 64, False, reps=10)
                res.update(n=n, uplo=uplo, transr=transr)
                rows.append(res)
    out["c2"] = {"workload": "config 2: n in {4000,4001} x 8 RFP variants, pftrf and pftrs(64) "
                             "(median of 10)", "variants": rows}
    # config 5: complex n=24000 'C' L pftrf -> pftri
    n = 24000
    a = spd(n, "1/n", True, seed=5)
    r = convert.trttf(a, "L", "C")
    pristine = r.data.clone()
    ts_f, ts_i = [], []
    for rep in range(2):
        r.data.copy_(pristine)
        s0, s1, s2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        s0.record()
        assert lib.rfpk_zpftrf(b"C", b"L", n, r.data.data_ptr(), info.data_ptr(), sh()) == 0
        s1.record()
        assert lib.rfpk_zpftri(b"C", b"L", n, r.data.data_ptr(), info.data_ptr(), sh()) == 0
        s2.record()
        s2.synchronize()
        assert int(info.item()) == 0
        ts_f.append(s0.elapsed_time(s1))
        ts_i.append(s1.elapsed_time(s2))
    del pristine
    J = torch.from_numpy(np.random.default_rng(11).choice(n, 256, replace=False)).to(dev)
    full = convert.tfttr(r)
    del r
    low, up = full[:, J], full[J, :].conj().t()
    Y = torch.where(torch.arange(n, device=dev).unsqueeze(1) >= J.unsqueeze(0), low, up)
    del full, low, up
    E = a @ Y
    E[J, torch.arange(256, device=dev)] -= 1.0
    tf, ti = min(ts_f), min(ts_i)
    out["c5"] = {"workload": "config 5: complex128 n=24000 TRANSR=C UPLO=L pftrf -> pftri (best of 2)",
                 "pftrf_ms": tf, "pftri_ms": ti, "pftrf_tflops": 4 * n ** 3 / 3 / tf / 1e9,
                 "pftri_tflops": 8 * n ** 3 / 3 / ti / 1e9,
                 "chain_tflops": 4 * n ** 3 / (tf + ti) / 1e9,
                 "chain_frac_nominal": 4 * n ** 3 / (tf + ti) / 1e9 / NOMINAL_FP64_TFLOPS,
                 "max_abs_AY_minus_I_256cols": float(E.abs().max())}
    del a, E, Y
    torch.cuda.empty_cache()
    # conversions at config 3's order, real (HBM roofline)
    n = C3_N
    nt = n * (n + 1) // 2
    src = torch.randn(n, n, dtype=torch.float64, device=dev)
    arf = torch.empty(nt, dtype=torch.float64, device=dev)
    pk = torch.empty(nt, dtype=torch.float64, device=dev)
    full = torch.empty(n, n, dtype=torch.float64, device=dev)
    conv = []
    for uplo in "LU":
        for transr in "NT":
            T, U = transr.encode(), uplo.encode()
            for name, fn, byts in (
                    ("trttf", lambda: lib.rfpk_dtrttf(T, U, n, src.data_ptr(), n, arf.data_ptr(), sh()), 2 * nt * 8),
                    ("tfttr", lambda: lib.rfpk_dtfttr(T, U, n, arf.data_ptr(), full.data_ptr(), n, sh()), (nt + n * n) * 8),
                    ("tfttp", lambda: lib.rfpk_dtfttp(T, U, n, arf.data_ptr(), pk.data_ptr(), sh()), 2 * nt * 8),
                    ("tpttf", lambda: lib.rfpk_dtpttf(T, U, n, pk.data_ptr(), arf.data_ptr(), sh()), 2 * nt * 8)):
                ms = ev_time(fn, 5)
                gbs = byts / (ms * 1e-3) / 1e9
                conv.append({"op": name, "uplo": uplo, "transr": transr, "ms": ms, "gbs": gbs,
                             "frac_hbm": gbs / hbm_peak()})
    out["conversions"] = {"workload": f"real n={n}: trttf/tfttr/tfttp/tpttf, 4 layouts (median of 5); "
                                      "bytes = every element read once and written once (tfttr "
                                      "also writes the zeroed other triangle)",
                          "peak_gbs": hbm_peak(), "ops": conv}
    del src, arf, pk, full
    torch.cuda.empty_cache()
    return out


# ---------------------------------------------------------------- main
def run_b200(args, rank, world, local):
    import torch
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    line = run_c3(args, rank, world, local)
    torch.cuda.empty_cache()
    if not args.no_batched:
        line["batched"] = run_c4(args, rank, world, local)
        torch.cuda.empty_cache()
    if rank != 0:
        return
    if world == 1 and not args.no_configs:
        line["per_config"] = per_config(dev)
    if world == 1 and not args.no_cpu:
        line["cpu_baseline"] = cpu_baseline_c3()
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--batch", type=int, default=65536)
    ap.add_argument("--no-cpu", action="store_true", help="skip the full-size reference leg")
    ap.add_argument("--no-configs", action="store_true", help="skip the per_config blocks")
    ap.add_argument("--no-batched", action="store_true", help="skip the config-4 block")
    ap.add_argument("--no-e2e", action="store_true", help="skip the host-buffer legs (profiling)")
    args = ap.parse_args()
    if args.impl == "b200":
        args.warmup = max(3, args.warmup)  # the contract's minimum; the line reports it
    if int(os.environ.get("WORLD_SIZE", "1")) > 1:
        os.environ.setdefault("NCCL_DEBUG", "INFO")  # communicator lines show the N ranks
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    if args.impl == "reference":
        # rank 0 alone times the CPU path; the other ranks exit 0 without work
        # (no process group: nothing here is collective)
        rank, world, _ = dist_env()
        run_reference(args, rank, world)
        return
    rank, world, local = dist_setup()
    run_b200(args, rank, world, local)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
