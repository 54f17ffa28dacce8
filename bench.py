#!/usr/bin/env python
"""Benchmark contract for the B200 RFPF path ("Measurement").

Default workload = BASELINE config 3 (the north-star target): one real FP64
SPD matrix, n = 16384, TRANSR='N', UPLO='L', A = B B^T / n + I; a step is
pftrf followed by pftrs with nrhs = 1024, on an RFP buffer restored from a
pristine device copy at the start of the step (the RFP buffer, 1.07 GB, and
the RHS exceed the 126 MB L2, so no flush is needed).  Metric: FP64 GFLOP/s
with the LAPACK flop model n^3/3 + 2 n^2 nrhs.

  python bench.py [--gpus N --steps K --warmup W] [--impl reference]
  --workload c3 (default) | c4   (c1, c2, c5: tools/perf.py, tools/config5.py)

Under torchrun (N > 1) every rank factors its own replica (single matrices
do not shard: "replicas only", weak scaling); config 4 (--workload c4) is
sharded by matrix.  --impl reference times the reference's own CPU path
(the unmodified `rfpk` package installed into baseline/_ref from
/root/reference/pkg; falls back to the NumPy oracle port if absent) on a
bounded sample of the same workload on the host cores.
"""

from __future__ import annotations

import argparse
import ctypes
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


def ncu_traffic(key):
    """DRAM bytes per launch of a kernel from a committed ncu --set full
    capture (profiles/ncu_traffic.json), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            return json.load(f)[key]["bytes"]
    except Exception:
        return None


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except Exception:
        return {}


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
def dist_setup(n_gpus):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        import torch
        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
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
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ---------------------------------------------------------------- CPU baselines
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


def cpu_sample(n=4096, nrhs=256, reps=2, seed=3):
    """pftrf + pftrs on the host cores on a bounded sample of config 3: the
    reference itself (baseline/_ref, kind "reference") when installed, else
    the oracle port (kind "port")."""
    from oracle import rfp_oracle as O
    ref = _reference_module()
    a = O.spd_matrix(n, seed, "1/n")
    b0 = np.asfortranarray(np.random.default_rng(seed + 1).standard_normal((n, nrhs)))
    ts = []
    for _ in range(reps):
        x = b0.copy(order="F")
        if ref is not None:
            r = ref.convert.trttf(a, "L", "N")
            t0 = time.perf_counter()
            assert ref.rfp.pftrf(r) == 0
            ref.rfp.pftrs(r, x)
        else:
            buf = O.trttf(a, "L", "N")
            t0 = time.perf_counter()
            assert O.pftrf(buf, n, "L", "N") == 0
            O.pftrs(buf, n, "L", "N", x)
        ts.append(time.perf_counter() - t0)
    cores = _threads()
    flops = n ** 3 / 3 + 2 * n * n * nrhs
    t = float(np.median(ts))
    who = "reference rfpk (baseline/_ref)" if ref is not None else "oracle port"
    return {"value": flops / t / 1e9, "unit": "GFLOP/s", "cores": cores,
            "kind": "reference" if ref is not None else "port",
            "sample": f"{who} pftrf+pftrs n={n} LN nrhs={nrhs} (median of {reps}, "
                      f"{t:.2f} s each; numpy/OpenBLAS {cores} threads)"}


def c3_config(n, nrhs, world):
    return {"workload": "BASELINE config 3: pftrf+pftrs, n=16384, TRANSR=N, UPLO=L, nrhs=1024",
            "n": n, "nrhs": nrhs, "transr": "N", "uplo": "L",
            "l2": "no flush: RFP buffer 1.07 GB + RHS 134 MB exceed the 126 MB L2",
            "call": "rfpk_dpfsv (pftrf + pftrs in one C-ABI call; e2e: rfpk_dpfsv_host)",
            "parallelism": "replicas" if world > 1 else "single GPU"}


def c4_config(total, n, nrhs, world):
    return {"workload": "BASELINE config 4: 65536 x n=64 UN pftrf+pftrs(nrhs=8), sharded by matrix",
            "batch": total, "n": n, "nrhs": nrhs, "parallelism": f"dp{world} (contiguous shards)",
            "l2": "no flush: every step factors its own fresh 1.6 GB copy"}


def _batched_worker(args):
    """One process's share of the reference's batched sample (single-threaded
    BLAS, as SURVEY 8(d) prescribes for config 4)."""
    first, count = args
    from threadpoolctl import threadpool_limits
    with threadpool_limits(1):
        return cpu_sample_batched(count=count, first=first)["value"]


def run_reference_c4(args, rank, world):
    """Reference arm for config 4: the reference's own pftrf+pftrs on n=64
    matrices, one process per host core (each single-threaded), a bounded
    sample of the 65,536 per step."""
    import concurrent.futures as cf
    cores = _threads()
    per = 48
    steps = []
    with cf.ProcessPoolExecutor(max_workers=cores) as ex:
        for i in range(args.warmup + args.steps):
            t0 = time.perf_counter()
            list(ex.map(_batched_worker, [(1000 * i + c * per, per) for c in range(cores)]))
            t = time.perf_counter() - t0
            if i >= args.warmup:
                steps.append(cores * per / t)
    value = float(np.mean(steps))
    kind = "reference" if _reference_module() is not None else "port"
    line = {
        "impl": "reference", "metric": METRIC_C4, "value": value, "unit": "matrices/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": cores * per / value * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded numpy)",
        "config": c4_config(args.batch, 64, 8, world),
        "cpu_baseline": {"value": value, "unit": "matrices/s", "cores": cores, "kind": kind,
                         "sample": f"{cores} processes x {per} matrices n=64 UN pftrf+pftrs(8) per "
                                   f"step, single-threaded BLAS each"},
        "e2e": {"value": value, "unit": "matrices/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_reference(args, rank, world):
    if rank != 0:
        return
    if args.workload == "c4":
        return run_reference_c4(args, rank, world)
    steps = []
    res = None
    for i in range(args.warmup + args.steps):
        res = cpu_sample(n=args.ref_n, nrhs=args.ref_nrhs, reps=1, seed=3 + i)
        if i >= args.warmup:
            steps.append(res["value"])
    value = float(np.mean(steps))
    n, nrhs = 16384, 1024
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "GFLOP/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": (args.ref_n ** 3 / 3 + 2 * args.ref_n ** 2 * args.ref_nrhs) / value / 1e6,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded numpy)",
        "config": c3_config(n, nrhs, world),
        "cpu_baseline": {"value": value, "unit": "GFLOP/s", "cores": res["cores"],
                         "kind": res["kind"], "sample": res["sample"]},
        "e2e": {"value": value, "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


METRIC = "FP64 GFLOP/s of RFPF pftrf+pftrs (n=16384, TRANSR=N, UPLO=L, nrhs=1024)"


# ---------------------------------------------------------------- GPU arm
def run_b200(args, rank, world, local):
    import torch
    from paper_0901_1696_b200 import _capi, convert, rfp
    from paper_0901_1696_b200.layout import make_descriptor

    lib = _capi.lib()
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    n, nrhs, uplo, transr = args.n, args.nrhs, "L", "N"
    desc = make_descriptor(n, uplo, transr)
    flops = n ** 3 / 3 + 2 * n * n * nrhs

    # inputs: B ~ N(0,1) seeded on the host, A = B B^T / n + I formed on the device
    seed = 1234 + rank
    rng = np.random.default_rng(seed)
    bh = torch.from_numpy(rng.standard_normal((n, n)))
    bd = bh.to(dev)
    del bh
    a = bd @ bd.t()
    a /= n
    a.diagonal().add_(1.0)
    del bd
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
        # pftrf + pftrs in one C-ABI call (rfpk_dpfsv: the first T1 solve and
        # the S1 product run beside potrf(T2)); the same work as the pair
        rc = lib.rfpk_dpfsv(T, U, n, nrhs, work.data_ptr(), x.data_ptr(), n, info.data_ptr(), sh)
        if rc:
            raise RuntimeError(f"rfpk call failed rc={rc}")

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    assert int(info.item()) == 0, "factorization failed"

    barrier(world)
    torch.cuda.synchronize()
    l0 = lib.rfpk_launch_count()
    lib.rfpk_phase_clock(1)  # event pairs around the SRPA steps, read after the loop
    with ClockSampler(local) as clk:
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(st)
        for _ in range(args.steps):
            step()
        e.record(st)
        torch.cuda.synchronize()
    launches = lib.rfpk_launch_count() - l0
    live_ms, live_n = ctypes.c_double(0.0), ctypes.c_int64(0)
    lib.rfpk_phase_time(b"pftrf syrk(T2)", ctypes.byref(live_ms), ctypes.byref(live_n))
    lib.rfpk_phase_clock(0)
    kms_live = live_ms.value / live_n.value if live_n.value else None
    barrier(world)
    ms = max_over_ranks(s.elapsed_time(e) / args.steps, world)
    value = world * flops / (ms * 1e-3) / 1e9

    # result check: ||A X - B|| / (||A|| ||X|| n eps) on the last step's solution
    r = a @ x - rhs0
    resid = float(r.norm() / (a.norm() * x.norm() * n * 2.0 ** -53))

    # dominant kernel: the largest launch that runs on its own inside the step,
    # pftrf's SYRK T2 <- T2 - S1 S1^T (gemm_kernel TRI: the 8192 x 8192 lower
    # triangle of a rank-8192 update, ~25% of the step).  (The S1 solve,
    # tile_trsm_kernel, is as long but now runs concurrently with potrf(T1) --
    # potrf_trsm_overlap -- so no single-kernel duration exists for it inside
    # the step.)  Timed live by the phase clock; alone through the C ABI on
    # the live RFP views, CUDA events on the launch stream, as a cross-check.
    ld = desc.ldar
    kern_flops = desc.n2 * desc.n2 * desc.n1  # n^2 k for the triangle of a rank-k update
    t2p = work.data_ptr()
    s1p = work.data_ptr() + 8 * (desc.n1 + desc.shift)

    def dom():
        lib.rfpk_dsyrk(b"U", b"C", -1.0, s1p, desc.n2, desc.n1, 1, ld, 1.0, t2p, desc.n2, 1, ld,
                       sh)

    dom()
    torch.cuda.synchronize()
    ks, ke = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    kreps = 3
    ks.record(st)
    for _ in range(kreps):
        dom()
    ke.record(st)
    torch.cuda.synchronize()
    kms_alone = ks.elapsed_time(ke) / kreps
    # achieved = flops per launch / the launch's average duration measured
    # live over the timed region (phase clock); the standalone timing is the
    # cross-check
    kms = kms_live if kms_live else kms_alone
    k_tflops = kern_flops / (kms * 1e-3) / 1e12

    # measured DGEMM ceiling (cuBLAS via torch) for context
    g1 = torch.randn(8192, 8192, dtype=torch.float64, device=dev)
    g2 = torch.randn(8192, 8192, dtype=torch.float64, device=dev)
    torch.matmul(g1, g2)
    torch.cuda.synchronize()
    gs, ge = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    gs.record(st)
    for _ in range(3):
        torch.matmul(g1, g2)
    ge.record(st)
    torch.cuda.synchronize()
    dgemm_tflops = 3 * 2 * 8192 ** 3 / (gs.elapsed_time(ge) * 1e-3) / 1e12
    del g1, g2

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
        r_, inf = rfp.pfsv_from_host(host_rfp, host_b.t(), n, uplo, transr, out=out_x.t())
        assert inf == 0

    e2e_step()
    barrier(world)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    es, ee = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    es.record(st)
    for _ in range(e2e_steps):
        e2e_step()
    ee.record(st)
    torch.cuda.synchronize()
    e2e_ms = max_over_ranks(es.elapsed_time(ee) / e2e_steps, world)
    e2e_value = world * flops / (e2e_ms * 1e-3) / 1e9

    if rank != 0:
        return
    cpu = cpu_sample() if (world == 1 and not args.no_cpu) else None
    line = {
        "metric": METRIC, "value": value, "unit": "GFLOP/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic: B~N(0,1) seeded numpy, A=B B^T/n+I (formed on device), RHS~N(0,1)",
        "config": c3_config(n, nrhs, world),
        "fraction_of_fp64_nominal": value / 1e3 / NOMINAL_FP64_TFLOPS,
        "fraction_of_fp64_measured_dgemm": value / 1e3 / dgemm_tflops,
        "roofline": {"bound": "tensor",
                     "kernel": "gemm_kernel TRI (pftrf SYRK T2 -= S1 S1^T: 8192x8192 lower triangle, k=8192)",
                     "achieved": k_tflops, "peak": NOMINAL_FP64_TFLOPS, "unit": "TFLOP/s",
                     "frac": k_tflops / NOMINAL_FP64_TFLOPS,
                     "algorithmic_flops": kern_flops, "ms_per_launch": kms,
                     "timing": ("live: CUDA events around the launch inside every timed step "
                                f"({live_n.value} launches); alone: {kms_alone:.3f} ms")
                     if kms_live else "standalone launch (phase clock unavailable)",
                     "traffic": ncu_traffic("syrk_T2_n16384_LN"),
                     "algorithmic_bytes": 8 * (desc.n1 * desc.n2 + desc.n2 * (desc.n2 + 1)),
                     "peak_source": "nominal FP64 DMMA (MEASURED_PEAKS.json has no FP64 figure); "
                                    f"measured cuBLAS DGEMM here: {dgemm_tflops:.2f} TFLOP/s"},
        "residual_scaled": resid,
        "e2e": {"value": e2e_value, "unit": "GFLOP/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "ms_per_step": e2e_ms,
                "path": "rfp.pfsv_from_host (public API): pinned host RFP + RHS in, solution out, transfers overlapped with pftrf/pftrs"},
        "gpu_launches": launches,
        "clocks": clk.summary(),
    }
    if cpu:
        line["cpu_baseline"] = cpu
    print(json.dumps(line), flush=True)


METRIC_C4 = "matrices/s of batched RFPF pftrf+pftrs (65536 x n=64, TRANSR=N, UPLO=U, nrhs=8)"


def rfp_gather_index(n, uplo, transr):
    """For every RFP slot, the column-major offset i + j*n of the triangle
    element it holds (from the product's layout module, not the oracle)."""
    from paper_0901_1696_b200.layout import make_descriptor, map_index
    d = make_descriptor(n, uplo, transr)
    idx = np.empty(d.nt, dtype=np.int64)
    for j in range(1, n + 1):
        for i in (range(j, n + 1) if uplo == "L" else range(1, j + 1)):
            idx[map_index(d, i, j) - 1] = (i - 1) + (j - 1) * n
    return idx


def make_c4_inputs(start, stop, n, nrhs, seed0, dev):
    """A_k = B_k B_k^T + n I with B_k ~ N(0,1) from default_rng(seed0 + k)
    (BASELINE config 4), right-hand sides from default_rng(seed0 + 10**7 + k);
    returns (full A (count, n, n), RFP (count, nt), B (count, n, nrhs) col-major)."""
    import torch
    count = stop - start
    bh = np.empty((count, n, n))
    rh = np.empty((count, nrhs, n))
    for k in range(count):
        bh[k] = np.random.default_rng(seed0 + start + k).standard_normal((n, n))
        rh[k] = np.random.default_rng(seed0 + 10 ** 7 + start + k).standard_normal((nrhs, n))
    bd = torch.from_numpy(bh).to(dev)
    a = torch.bmm(bd, bd.transpose(1, 2))
    a.diagonal(dim1=1, dim2=2).add_(float(n))
    del bd
    idx = torch.from_numpy(rfp_gather_index(n, "U", "N")).to(dev)
    arf = a.transpose(1, 2).reshape(count, n * n)[:, idx].contiguous()  # column-major gather
    rhs = torch.from_numpy(rh).to(dev).transpose(1, 2)  # (count, n, nrhs) column-major
    return a, arf, rhs


def run_c4(args, rank, world, local):
    """Config 4: 65,536 independent n=64 matrices sharded by contiguous ranges;
    one fused batched launch per step per rank; the only collective is the
    NCCL gather of per-matrix (info, residual) after the timed region."""
    import torch
    from paper_0901_1696_b200 import _capi
    from paper_0901_1696_b200.shard import gather_results, shard_range

    lib = _capi.lib()
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    total, n, nrhs = args.batch, 64, 8
    start, stop = shard_range(total, rank, world)
    count = stop - start
    nt = n * (n + 1) // 2
    a, arf0, rhs0 = make_c4_inputs(start, stop, n, nrhs, 20260000, dev)
    nbuf = args.warmup + args.steps
    # every step factors a fresh copy (no restore inside the timed region, and
    # 1.6 GB per step keeps every step out of L2)
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

    for i in range(args.warmup):
        step(i)
    torch.cuda.synchronize()
    barrier(world)
    torch.cuda.synchronize()
    l0 = lib.rfpk_launch_count()
    with ClockSampler(local) as clk:
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(st)
        for i in range(args.warmup, nbuf):
            step(i)
        e.record(st)
        torch.cuda.synchronize()
    launches = lib.rfpk_launch_count() - l0
    ms = max_over_ranks(s.elapsed_time(e) / args.steps, world)
    value = total / (ms * 1e-3)

    # per-matrix scaled residual ||A x - b||_max / (||A||_max ||x||_max n eps), then gather
    x = rhss[-1]
    r = torch.bmm(a, x) - rhs0
    resid = r.abs().amax(dim=(1, 2)) / (a.abs().amax(dim=(1, 2)) * x.abs().amax(dim=(1, 2)) * n * 2.0 ** -53)
    torch.cuda.synchronize()
    g0 = time.perf_counter()
    gi, gr = gather_results(info, resid, total) if world > 1 else (info, resid)
    torch.cuda.synchronize()
    gather_ms = (time.perf_counter() - g0) * 1e3

    # e2e through the public API with pinned host buffers
    from paper_0901_1696_b200 import rfp
    host_arf = arf0.cpu().pin_memory()
    host_b = rhs0.transpose(1, 2).contiguous().cpu().pin_memory()  # (count, nrhs, n)
    out_b = torch.empty_like(host_b).pin_memory()

    def e2e_step():
        # one public call: the chunked host pipeline (copies in and out
        # overlapped with the fused kernel; rfp.pftrf_pftrs_batched_from_host)
        _, inf = rfp.pftrf_pftrs_batched_from_host(host_arf, "N", "U", n, host_b.transpose(1, 2),
                                                   out=out_b.transpose(1, 2))
        torch.cuda.current_stream().synchronize()
        return inf

    e2e_step()
    barrier(world)
    es, ee = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e2e_steps = max(1, args.steps // 2)
    es.record(st)
    for _ in range(e2e_steps):
        e2e_step()
    ee.record(st)
    torch.cuda.synchronize()
    e2e_ms = max_over_ranks(es.elapsed_time(ee) / e2e_steps, world)
    if rank != 0:
        return
    per_matrix_bytes = 2 * nt * 8 + 2 * n * nrhs * 8
    hbm_peak = float(peaks().get("hbm_gbs", 6525.6))
    achieved_gbs = total / world * per_matrix_bytes / (ms * 1e-3) / 1e9 if world == 1 else \
        count * per_matrix_bytes / (ms * 1e-3) / 1e9
    cpu = None
    if world == 1 and not args.no_cpu:
        cpu = cpu_sample_batched()
    line = {
        "metric": METRIC_C4, "value": value, "unit": "matrices/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic: B_k~N(0,1) from default_rng(seed0+k), A_k=B_k B_k^T+64 I",
        "config": c4_config(total, n, nrhs, world),
        "roofline": {"bound": "hbm", "kernel": "batched64_kernel (fused pftrf+pftrs)",
                     "achieved": achieved_gbs, "peak": hbm_peak, "unit": "GB/s",
                     "frac": achieved_gbs / hbm_peak,
                     "traffic": ncu_traffic("batched64_fused_65536") if count == 65536 else None,
                     "bytes_per_matrix": per_matrix_bytes},
        "max_residual_scaled": float(gr.max()), "failed_matrices": int((gi != 0).sum()),
        "gather_ms": gather_ms,
        "e2e": {"value": total / (e2e_ms * 1e-3), "unit": "matrices/s",
                "h2d_bytes_per_step": host_arf.numel() * 8 + host_b.numel() * 8,
                "d2h_bytes_per_step": host_b.numel() * 8, "ms_per_step": e2e_ms},
        "gpu_launches": launches, "clocks": clk.summary(),
    }
    if cpu:
        line["cpu_baseline"] = cpu
    print(json.dumps(line), flush=True)


def cpu_sample_batched(count=256, n=64, nrhs=8, first=0):
    """Reference (or oracle) pftrf+pftrs on `count` n=64 UN matrices, one
    process, BLAS single-threaded semantics are the reference's own."""
    from oracle import rfp_oracle as O
    ref = _reference_module()
    mats = [O.spd_matrix(n, first + k, "n") for k in range(count)]
    rhs = [np.asfortranarray(np.random.default_rng(first + k).standard_normal((n, nrhs)))
           for k in range(count)]
    t0 = time.perf_counter()
    for a, b in zip(mats, rhs):
        x = b.copy(order="F")
        if ref is not None:
            r = ref.convert.trttf(a, "U", "N")
            ref.rfp.pftrf(r)
            ref.rfp.pftrs(r, x)
        else:
            buf = O.trttf(a, "U", "N")
            O.pftrf(buf, n, "U", "N")
            O.pftrs(buf, n, "U", "N", x)
    t = time.perf_counter() - t0
    return {"value": count / t, "unit": "matrices/s", "cores": 1,
            "kind": "reference" if ref is not None else "port",
            "sample": f"{count} matrices n=64 UN pftrf+pftrs(8) in one process ({t:.2f} s; "
                      f"trttf excluded)"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--n", type=int, default=16384)
    ap.add_argument("--nrhs", type=int, default=1024)
    ap.add_argument("--ref-n", type=int, default=4096)
    ap.add_argument("--ref-nrhs", type=int, default=256)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--workload", default="c3", choices=["c3", "c4"])
    ap.add_argument("--batch", type=int, default=65536)
    args = ap.parse_args()
    rank, world, local = dist_setup(args.gpus)
    if args.impl == "reference":
        run_reference(args, rank, world)
    elif args.workload == "c4":
        run_c4(args, rank, world, local)
    else:
        run_b200(args, rank, world, local)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
