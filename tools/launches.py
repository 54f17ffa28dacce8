"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list."""
import csv, re, sys
from collections import defaultdict
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]; rows = rows[1:]
ki = hdr.index("Kernel Name"); vi = hdr.index("Metric Value"); ui = hdr.index("Metric Unit")
agg = defaultdict(lambda: [0, 0.0])
tot = 0.0
for r in rows:
    v = float(r[vi].replace(",", "")); u = r[ui]
    us = v / 1000 if u in ("nsecond", "ns") else (v if u == "usecond" else v * 1000)
    name = r[ki]
    base = re.sub(r"^void ", "", name).replace("<unnamed>::", "").split("(")[0].split("<")[0]
    key = base.split("::")[-1] or name[:40]
    if "gemm" in key:
        t = re.search(r"<(\d+), (\d+), (\d+),", name)
        key += f"<{t.group(1)}x{t.group(2)}>" if t else ""
        key += " TRI" if re.search(r"\(int\)[12]>|, [12]>", name) else ""
    agg[key][0] += 1; agg[key][1] += us; tot += us
print(f"total {tot/1000:.2f} ms over {len(rows)} launches")
for k, (c, us) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{us/1000:9.3f} ms {100*us/tot:5.1f}%  n={c:5d}  avg={us/c:8.1f} us  {k}")
