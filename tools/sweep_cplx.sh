for v in 0 1; do
  echo "== RFPK_TRTRI_OOP_CPLX=$v"
  for n in 1000 2000 6000 8000; do
    RFPK_TRTRI_OOP_CPLX=$v python - <<PY
import sys; sys.argv=['x']; sys.path.insert(0,'tools'); import perf
perf.rfp_bench($n, "L", "T", 0, do_pftri=True, cplx=True, reps=3)
PY
  done
done
