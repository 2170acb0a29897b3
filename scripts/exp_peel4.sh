mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launch_k4.csv python scripts/run_tc.py --config C4 --reps 1 --what analysis --k 4 > gpurun_out/launch_k4.log 2>&1; echo ncu rc=$?
GC_PEEL_TRACE=2 timeout 600 python scripts/run_tc.py --config C4 --reps 2 --what analysis --k 4 > gpurun_out/trace_k4.log 2>&1; echo trace rc=$?; tail -30 gpurun_out/trace_k4.log
