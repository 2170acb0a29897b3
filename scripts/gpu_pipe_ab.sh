# GC_OPT_PIPE check and A/B: oracle parity of the pipelined kernel, then C4 / C5 TC + support times
mkdir -p gpurun_out
timeout 600 python scripts/diag/pipe_check.py > gpurun_out/pipe_check.log 2>&1; echo pipe_check rc=$?; tail -3 gpurun_out/pipe_check.log
for o in 21=0 21=1 21=0 21=1; do
  echo "== C4 $o"; timeout 300 python scripts/run_tc.py --config C4 --reps 2 --what tc,support --opt $o 2>&1 | tail -1 | cut -c1-120
done
for o in 21=0 21=1; do
  echo "== C5 $o"; timeout 600 python scripts/run_tc.py --config C5 --reps 1 --what tc,support --opt $o 2>&1 | tail -1 | cut -c1-120
done
