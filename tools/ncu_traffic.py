"""Rebuild profiles/ncu_traffic.json from an ncu launch list of one bench step.

  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
      --clock-control none --csv --log-file profiles/rNN_ncu_step_launches.csv \
      python bench.py --steps 1 --warmup 3 --no-cpu --no-configs --no-batched --no-e2e
  python tools/ncu_traffic.py profiles/rNN_ncu_step_launches.csv

The library's kernels of the LAST bench step (the timed one) are the last
`per_step` rfpk launches; each is keyed by the kernel-clock label bench.py
uses (config 3: n1 = n2 = 8192, nrhs = 1024)."""
import csv
import json
import sys
from collections import defaultdict

src = sys.argv[1]
per_step = int(sys.argv[2]) if len(sys.argv) > 2 else 14
rows = [r for r in csv.reader(open(src)) if len(r) > 10]
hdr = rows[0]
ix = {h: i for i, h in enumerate(hdr)}
launch = defaultdict(dict)
names = {}
for r in rows[1:]:
    lid = int(r[ix["ID"]])
    names[lid] = r[ix["Kernel Name"]]
    v = float(r[ix["Metric Value"]].replace(",", ""))
    launch[lid][r[ix["Metric Name"]]] = v if r[ix["Metric Unit"]] not in ("nsecond", "ns") else v / 1e6
ours = [lid for lid in sorted(launch) if "rfpk::" in names[lid]]
# the step ends with pftrs's last narrow solve; what follows it (bench.py's
# standalone timing of the dominant kernel's largest launch) is not the step
end = len(ours)
while end > 0 and not ("tile_trsm_kernel" in names[ours[end - 1]] and
                       launch[ours[end - 1]].get("gpu__time_duration.sum", 0.0) < 8.0):
    end -= 1
step = ours[max(0, end - per_step):end]


def label(lid):
    nm, d = names[lid], launch[lid]
    ms = d.get("gpu__time_duration.sum", 0.0)
    if "tile_potrf_kernel" in nm:
        return "kernel tile_potrf 8192x8192"
    if "tile_trsm_kernel" in nm:
        return "kernel tile_trsm 8192x8192" if ms > 8.0 else "kernel tile_trsm 8192x1024"
    if "tile_copy_kernel" in nm:
        return "kernel tile_copy 8192x8192"
    if "gemm_kernel" in nm:
        return "kernel syrk 8192x8192x8192" if ms > 12.0 else "kernel gemm 8192x1024x8192"
    return "other " + nm.split("(")[0].replace("void ", "")[:80]


acc = defaultdict(lambda: {"bytes": 0.0, "read": 0.0, "write": 0.0, "ms_ncu": 0.0, "n": 0})
for lid in step:
    d = launch[lid]
    a = acc[label(lid)]
    a["read"] += d.get("dram__bytes_read.sum", 0.0)
    a["write"] += d.get("dram__bytes_write.sum", 0.0)
    a["ms_ncu"] += d.get("gpu__time_duration.sum", 0.0)
    a["n"] += 1
out = {"_note": ("DRAM bytes (dram__bytes_read.sum + dram__bytes_write.sum) per launch, keyed by "
                 "the library's kernel-clock label; averaged over the launches of one config-3 "
                 f"step. Source: {src} (the last {per_step} library launches = the timed step; "
                 "tools/ncu_traffic.py). Serialised, cold-cache per-launch times ('ms_ncu') are "
                 "for the share of the step, not absolute.")}
for k, a in sorted(acc.items(), key=lambda kv: -kv[1]["ms_ncu"]):
    n = a["n"]
    out[k] = {"bytes": (a["read"] + a["write"]) / n, "read": a["read"] / n,
              "write": a["write"] / n, "ms_ncu": a["ms_ncu"] / n, "launches_in_step": n}
# config 4's kernel: from the summary of its own `ncu --set full` capture
# (tools/ncu_summary.py prints the DRAM counters in GB)
import glob
import re
caps = sorted(glob.glob("profiles/r*_prof_batched_v*_summary.txt"),
              key=lambda f: [int(x) for x in re.findall(r"\d+", f)])
if caps:
    vals = dict(l.split()[:2] for l in open(caps[-1]) if l.startswith(("dram__", "gpu__time")))
    rd, wr = float(vals["dram__bytes_read.sum"]) * 1e9, float(vals["dram__bytes_write.sum"]) * 1e9
    out["kernel batched64 65536x8"] = {"bytes": rd + wr, "read": rd, "write": wr,
                                       "ms_ncu": float(vals["gpu__time_duration.sum"]),
                                       "launches_in_step": 1, "source": caps[-1]}
json.dump(out, open("profiles/ncu_traffic.json", "w"), indent=1)
tot = sum(a["ms_ncu"] for a in acc.values())
for k, a in sorted(acc.items(), key=lambda kv: -kv[1]["ms_ncu"]):
    print(f"{a['ms_ncu']:9.3f} ms {100 * a['ms_ncu'] / tot:5.1f}%  x{a['n']}  "
          f"{(a['read'] + a['write']) / a['n'] / 1e9:7.2f} GB/launch  {k}")
