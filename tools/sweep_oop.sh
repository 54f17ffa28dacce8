# pftri / tftri-heavy sizes with the one-launch forms off / default / always
for v in 0 4096 100000; do
  echo "== RFPK_OOP_MAX=$v"
  for n in 300 1000 2000 4000 8000 12000; do
    RFPK_OOP_MAX=$v python - <<PY
import sys; sys.argv=['x']; sys.path.insert(0,'tools'); import perf
perf.rfp_bench($n, "L", "N", 0, do_pftri=True, reps=3)
PY
  done
done
