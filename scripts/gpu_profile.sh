# round profile: bench line, ncu launch list of one C4 pass, ncu --set full of the TC pass kernels, decomposition timings
mkdir -p gpurun_out
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.log 2>&1; echo bench rc=$?; tail -1 gpurun_out/bench.log | cut -c1-300
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
   python scripts/run_tc.py --config C4 --reps 1 --what tc,support,ktruss > gpurun_out/ncu_launch.log 2>&1; echo ncu_list rc=$?
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_tc_ -c 3 -o gpurun_out/prof_tc_c4 -f \
   python scripts/run_tc.py --config C4 --reps 1 --what tc > gpurun_out/ncu_full.log 2>&1; echo ncu_full rc=$?
for C in C1 C3 C4 C5; do timeout 900 python scripts/run_decomp.py --config $C --tc 1 --ks 3,4,5,6 2>&1 | grep -v "^gen\|^mem" ; done > gpurun_out/decomp.log 2>&1; cat gpurun_out/decomp.log
