# GC_OPT_PIPE check and A/B: oracle parity of the pipelined kernel, then C4 / C5 TC + support times
mkdir -p gpurun_out
timeout 600 python scripts/diag/pipe_check.py > gpurun_out/pipe_check.log 2>&1; echo pipe_check rc=$?; tail -3 gpurun_out/pipe_check.log
for o in 21=0 21=1 21=0 21=1; do
  echo "== C4 $o"; timeout 300 python scripts/run_tc.py --config C4 --reps 2 --what tc,support --opt $o 2>&1 | tail -1 | cut -c1-120
done
for o in 21=0 21=1; do
  echo "== C5 $o"; timeout 600 python scripts/run_tc.py --config C5 --reps 1 --what tc,support --opt $o 2>&1 | tail -1 | cut -c1-120
done
# peel: both survivor decrements in flight (tree) against the previous build (VAR)
for L in build_var/${VAR:-predec2}/libgc.so ""; do
  echo "== peel ${L:-tree}"
  GC_LIB_PATH=$L timeout 300 python scripts/run_tc.py --config C4 --reps 3 --what analysis --k 4 2>&1 | tail -1 | cut -c1-160
  GC_LIB_PATH=$L timeout 600 python scripts/run_decomp.py --config C4 2>&1 | tail -1
done
