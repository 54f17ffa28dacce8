"""GPU calibration probe (run under gpurun): FP64 mma fragment layouts,
DMMA/DFMA issue rates, cuBLAS DGEMM ceiling and cuSOLVER potrf comparator.

Writes one JSON object to stdout; nothing here is a bench number.
"""
import ctypes
import json
import os
import subprocess
import time

import numpy as np
import torch

here = os.path.dirname(os.path.abspath(__file__))
lib = ctypes.CDLL(os.path.join(here, "probe_mma.so"))
out = {}
dev = torch.device("cuda:0")
out["gpu"] = torch.cuda.get_device_name(0)

shapes = {0: (8, 8, 4), 1: (16, 8, 4), 2: (16, 8, 8), 3: (16, 8, 16)}
names = {0: "m8n8k4", 1: "m16n8k4", 2: "m16n8k8", 3: "m16n8k16"}
for w, (m, n, k) in shapes.items():
    A = torch.randn(m, k, dtype=torch.float64, device=dev)
    B = torch.randn(k, n, dtype=torch.float64, device=dev)
    D = torch.zeros(m, n, dtype=torch.float64, device=dev)
    rc = lib.launch_probe(w, ctypes.c_void_p(A.data_ptr()), ctypes.c_void_p(B.data_ptr()),
                          ctypes.c_void_p(D.data_ptr()))
    ref = A @ B
    out["layout_" + names[w]] = {"rc": rc, "maxerr": float((D - ref).abs().max())}


def rate(which, blocks, threads, iters):
    buf = torch.zeros(blocks * threads, dtype=torch.float64, device=dev)
    lib.launch_rate(which, ctypes.c_void_p(buf.data_ptr()), blocks, threads, iters)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    lib.launch_rate(which, ctypes.c_void_p(buf.data_ptr()), blocks, threads, iters)
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e)
    if which == 0:
        flop = blocks * (threads // 32) * iters * 16 * (16 * 8 * 4 * 2)
    else:
        flop = blocks * threads * iters * 16 * 2
    return flop / ms / 1e9


out["dmma_tflops"] = {f"{b}x{t}": rate(0, b, t, 2000) for b, t in [(148, 256), (148, 512), (296, 256)]}
out["dfma_tflops"] = {f"{b}x{t}": rate(1, b, t, 4000) for b, t in [(148, 512), (296, 512), (592, 256)]}

smi = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active",
                        "--format=csv,noheader", "-lms", "200"], stdout=subprocess.PIPE, text=True)


def timeit(fn, reps):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


for n in (4096, 8192):
    a = torch.randn(n, n, dtype=torch.float64, device=dev)
    b = torch.randn(n, n, dtype=torch.float64, device=dev)
    c = torch.empty(n, n, dtype=torch.float64, device=dev)
    ms = timeit(lambda: torch.matmul(a, b, out=c), 5)
    out[f"cublas_dgemm_{n}_tflops"] = 2 * n ** 3 / ms / 1e9
# sustained: 4 s of back-to-back DGEMM 8192
t0 = time.time()
cnt = 0
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
while time.time() - t0 < 4:
    torch.matmul(a, b, out=c)
    cnt += 1
    if cnt % 8 == 0:
        torch.cuda.synchronize()
e.record()
torch.cuda.synchronize()
out["cublas_dgemm_8192_sustained_tflops"] = cnt * 2 * 8192 ** 3 / s.elapsed_time(e) / 1e9

for n in (1000, 4000, 16384):
    g = torch.randn(n, n, dtype=torch.float64, device=dev)
    A = g @ g.T / n + torch.eye(n, dtype=torch.float64, device=dev)
    ms = timeit(lambda: torch.linalg.cholesky(A), 3)
    out[f"cusolver_potrf_{n}_ms"] = ms
    out[f"cusolver_potrf_{n}_tflops"] = n ** 3 / 3 / ms / 1e9
smi.terminate()
lines = smi.communicate()[0].strip().splitlines()
out["clocks_samples"] = lines[-20:]
out["cpu_count"] = os.cpu_count()
try:
    out["cpu_model"] = [l for l in open("/proc/cpuinfo") if "model name" in l][0].split(":")[1].strip()
except Exception:
    pass
print(json.dumps(out, indent=1))
