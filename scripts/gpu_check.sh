# round check: smoke, gpu tests, C4 bench line, ncu launch list
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv; nproc
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?; tail -2 gpurun_out/smoke.log
timeout 1200 python -m pytest tests -m gpu -x -q -p no:warnings > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -5 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.log 2>&1; echo bench rc=$?; tail -1 gpurun_out/bench.log | cut -c1-600
if [ "${PROF:-0}" = "1" ]; then
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
   python scripts/run_tc.py --config C4 --reps 1 --what tc,support,ktruss > gpurun_out/ncu_launch.log 2>&1; echo ncu_list rc=$?
fi
