# A/B of a variant build (VAR) against the in-tree libgc: C4 analysis(k=4) and C4/C5 decomposition times
for L in build_var/${VAR:-base}/libgc.so ""; do
  echo "== ${L:-tree}"
  GC_LIB_PATH=$L timeout 600 python scripts/run_tc.py --config C4 --reps 3 --what analysis --k 4 2>&1 | tail -1
  GC_LIB_PATH=$L timeout 600 python scripts/run_decomp.py --config C4 2>&1 | tail -1
  [ "${C5:-1}" = 1 ] && GC_LIB_PATH=$L timeout 900 python scripts/run_decomp.py --config C5 2>&1 | tail -1
done
