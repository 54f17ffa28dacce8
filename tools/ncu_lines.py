"""Per-source-line summary of an ncu --set full --import-source report.

usage: python tools/ncu_lines.py REPORT.ncu-rep [TOP]

Aggregates the CUDA-source view (`--page source --print-source cuda`) and
prints the lines with the most shared-memory wavefronts, the most executed
instructions and the most warp-stall samples."""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr_i = next(i for i, r in enumerate(rows) if any("Source" == c or c.startswith("# ") for c in r)
             or ("Source" in r))
hdr = rows[hdr_i]
body = [r for r in rows[hdr_i + 1:] if len(r) == len(hdr)]


def col(*subs):
    for i, h in enumerate(hdr):
        if all(s.lower() in h.lower() for s in subs):
            return i
    return None


def num(s):
    try:
        return float(s.replace(",", ""))
    except ValueError:
        return 0.0


src = col("source")
file_i = col("file") if col("file") is not None else None
line_i = col("line") if col("line") is not None else col("#")
wf = col("l1 wavefronts shared") if col("l1 wavefronts shared") is not None else col("wavefronts", "shared")
ins = col("instructions executed")
smp = col("warp stall sampling (all")
print("columns:", " | ".join(h for h in hdr[:40]))
tot = {k: sum(num(r[i]) for r in body) for k, i in (("wf", wf), ("ins", ins), ("smp", smp)) if i is not None}
print("totals:", tot)
for key, i in (("shared wavefronts", wf), ("instructions", ins), ("stall samples", smp)):
    if i is None:
        continue
    print(f"--- top by {key}")
    for r in sorted(body, key=lambda r: -num(r[i]))[:top]:
        vals = " ".join(f"{num(r[j]):>10.0f}" for j in (wf, ins, smp) if j is not None)
        loc = r[line_i] if line_i is not None else ""
        print(f"{vals}  {loc:>5}  {r[src].strip()[:90] if src is not None else ''}")
