# full round check: gpu tests, tune line, bench line, ncu launch list, ncu full capture of TC kernels
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:warnings > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/pytest_gpu.log
timeout 600 python scripts/tune.py C4 "block_batch=32" 2>&1 | tail -1
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.log 2>&1; echo bench rc=$?; tail -1 gpurun_out/bench.log | cut -c1-400
if [ "${PROF:-1}" = "1" ]; then
timeout 300 python scripts/run_tc.py --config C4 --reps 1 --what tc,support,ktruss > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
   python scripts/run_tc.py --config C4 --reps 1 --what tc,support,ktruss > gpurun_out/ncu_launch.log 2>&1; echo ncu_list rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_tc_ -c 6 -o gpurun_out/prof_tc_c4 -f \
   python scripts/run_tc.py --config C4 --reps 1 --what tc,support > gpurun_out/ncu_full.log 2>&1; echo ncu_full rc=$?
fi
