"""Per-source-line summary of an ncu --set full --import-source report.

usage: python tools/ncu_lines.py REPORT.ncu-rep [TOP]

Reads the mixed CUDA/SASS source view (`--page source --print-source
cuda,sass`): the source-line rows carry the metrics of their SASS, summed.
Prints totals per matrix-independent unit (whole launch), the lines with the
most shared-memory wavefronts, instructions and stall samples, and the SASS
opcode mix."""
import csv
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))


def num(s):
    try:
        return float(s.replace(",", ""))
    except ValueError:
        return 0.0


hdr = None
cur = ""
lines = []
ops = defaultdict(lambda: [0.0, 0.0])
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        ix = {h: i for i, h in enumerate(hdr)}
        WF, INS, SMP = ix["L1 Wavefronts Shared"], ix["Instructions Executed"], ix[
            "Warp Stall Sampling (All Samples)"]
        SRC2 = 3
        continue
    if hdr is None or len(r) != len(hdr):
        continue
    if r[0]:
        lines.append((num(r[WF]), num(r[INS]), num(r[SMP]), f"{cur}:{r[0]}", r[1].strip()))
    else:
        op = r[SRC2].split()[0] if r[SRC2].split() else "?"
        if op.startswith("@"):
            op = r[SRC2].split()[1]
        op = op.split(".")[0]
        ops[op][0] += num(r[INS])
        ops[op][1] += num(r[WF])

tot = [sum(x[i] for x in lines) for i in range(3)]
print(f"totals: shared wavefronts {tot[0]:.4g}  instructions {tot[1]:.4g}  samples {tot[2]:.4g}")
for key, i in (("shared wavefronts", 0), ("instructions", 1), ("stall samples", 2)):
    print(f"--- top by {key}   (wf  ins  samples  %samples)")
    for x in sorted(lines, key=lambda x: -x[i])[:top]:
        print(f"{x[0]:>11.0f} {x[1]:>11.0f} {x[2]:>7.0f} {100 * x[2] / max(tot[2], 1):5.1f}%  "
              f"{x[3]:<22} {x[4][:80]}")
print("--- SASS opcode mix (instructions, shared wavefronts)")
for op, (n, w) in sorted(ops.items(), key=lambda kv: -kv[1][0])[:20]:
    print(f"{op:<10} {n:>12.0f} {w:>12.0f}")
