# round-2 profile: bench line; one launch list (time + DRAM bytes per kernel) of a C4 build +
# TC pass + the step's gc_ktruss_analysis(4); ncu --set full of the support and TC block kernels
# and of the k = 4 peel's first round; a time + DRAM launch list of the C4 decomposition
mkdir -p gpurun_out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.log 2>&1; echo bench rc=$?; tail -1 gpurun_out/bench.log | cut -c1-200
timeout 900 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/launches.csv \
   python scripts/run_tc.py --config C4 --reps 1 --what tc,analysis --k 4 > gpurun_out/ncu_launch.log 2>&1; echo ncu_list rc=$?
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_tc_block -c 1 -o gpurun_out/r2_tc_block -f \
   python scripts/run_tc.py --config C4 --reps 1 --what tc > gpurun_out/ncu_full1.log 2>&1; echo ncu1 rc=$?
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_tc_block --launch-skip 1 -c 1 -o gpurun_out/r2_sup_block -f \
   python scripts/run_tc.py --config C4 --reps 1 --what tc,support > gpurun_out/ncu_full2.log 2>&1; echo ncu2 rc=$?
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_peel -c 1 -o gpurun_out/r2_peel_k4 -f \
   python scripts/run_tc.py --config C4 --reps 1 --what analysis --k 4 > gpurun_out/ncu_full3.log 2>&1; echo ncu3 rc=$?
timeout 1500 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/launches_decomp.csv \
   python scripts/run_decomp.py --config C4 > gpurun_out/ncu_decomp.log 2>&1; echo ncu_decomp rc=$?
