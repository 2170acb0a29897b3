# round profile: bench line, ncu launch list of one fused C4 step, per-kernel ncu --set full of the intersection kernels, decomposition timings
mkdir -p gpurun_out
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.log 2>&1; echo bench rc=$?; tail -1 gpurun_out/bench.log | cut -c1-200
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
   python scripts/run_tc.py --config C4 --reps 1 --what analysis > gpurun_out/ncu_launch.log 2>&1; echo ncu_list rc=$?
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_tc_block -c 1 -o gpurun_out/prof_tc_c4 -f \
   python scripts/run_tc.py --config C4 --reps 1 --what tc > gpurun_out/ncu_full1.log 2>&1; echo ncu1 rc=$?
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_tc_warp -c 1 -o gpurun_out/prof_tc_warp_c4 -f \
   python scripts/run_tc.py --config C4 --reps 1 --what tc > gpurun_out/ncu_full2.log 2>&1; echo ncu2 rc=$?
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_tc_tiny -c 1 -o gpurun_out/prof_tc_tiny_c4 -f \
   python scripts/run_tc.py --config C4 --reps 1 --what tc > gpurun_out/ncu_full3.log 2>&1; echo ncu3 rc=$?
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_tc_block --launch-skip 1 -c 1 -o gpurun_out/prof_sup_block_c4 -f \
   python scripts/run_tc.py --config C4 --reps 1 --what tc,support > gpurun_out/ncu_full4.log 2>&1; echo ncu4 rc=$?
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_tc_warp --launch-skip 1 -c 1 -o gpurun_out/prof_sup_warp_c4 -f \
   python scripts/run_tc.py --config C4 --reps 1 --what tc,support > gpurun_out/ncu_full5.log 2>&1; echo ncu5 rc=$?
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_tc_tiny --launch-skip 1 -c 1 -o gpurun_out/prof_sup_tiny_c4 -f \
   python scripts/run_tc.py --config C4 --reps 1 --what tc,support > gpurun_out/ncu_full6.log 2>&1; echo ncu6 rc=$?
for C in C1 C3 C4 C5 K13; do timeout 900 python scripts/run_decomp.py --config $C --tc 1 --ks 3,4,5,6 2>&1 | grep -v "^gen\|^mem" ; done > gpurun_out/decomp.log 2>&1; cat gpurun_out/decomp.log
