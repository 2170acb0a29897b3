# bench line + ncu launch list + full capture of the TC kernels (C4)
mkdir -p gpurun_out
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.log 2>&1; echo bench rc=$?; tail -1 gpurun_out/bench.log
timeout 300 python scripts/run_tc.py --config C4 --reps 1 --what tc,support,ktruss > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
   python scripts/run_tc.py --config C4 --reps 1 --what tc,support,ktruss > gpurun_out/ncu_launch.log 2>&1; echo ncu_list rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_tc_ -c 6 -o gpurun_out/prof_tc_c4 -f \
   python scripts/run_tc.py --config C4 --reps 1 --what tc,support > gpurun_out/ncu_full.log 2>&1; echo ncu_full rc=$?
