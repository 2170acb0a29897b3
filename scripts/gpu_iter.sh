# iteration check: selected GPU tests (PYTEST_K), then C4 build/pass times for option A/B (AB_OPTS)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -p no:warnings ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -4 gpurun_out/pytest_gpu.log
for o in ${AB_OPTS:-none}; do
  if [ "$o" = none ]; then a=""; else a="--opt $o"; fi
  echo "== $o"; timeout 600 python scripts/run_tc.py --config ${CFG:-C4} --reps 3 --what ${WHAT:-tc,analysis} --k 4 $a 2>&1 | tail -2
done
