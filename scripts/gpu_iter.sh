# iterate: gpu tests, C3/C4 phase timings, ncu launch list + full capture of the TC kernels at C4
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:warnings > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python scripts/run_tc.py --config C3 --reps 3 --what tc,support,ktruss 2>&1 | tail -2
timeout 300 python scripts/run_tc.py --config C4 --reps 3 --what tc,support,ktruss 2>&1 | tail -2
if [ "${NCU:-0}" = "1" ]; then
timeout 300 python scripts/run_tc.py --config C4 --reps 1 --what tc > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_tc_ -c 3 -o gpurun_out/prof_tc_c4 -f \
   python scripts/run_tc.py --config C4 --reps 1 --what tc > gpurun_out/ncu_full.log 2>&1; echo ncu rc=$?
fi
