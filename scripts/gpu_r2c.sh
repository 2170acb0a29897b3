mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_gpu.py -x -q -p no:warnings -k "uw_hit_bits or forced or heavy or huge or task_chunk or fuzz or golden or c3_full or large_clique" > gpurun_out/pytest_uw.log 2>&1; echo pytest rc=$?; tail -5 gpurun_out/pytest_uw.log
timeout 600 python scripts/tune.py C4 'uw_bits=1' 'uw_bits=0' 'uw_bits=1' 'uw_bits=0' > gpurun_out/tune_uw.log 2>&1; echo tune rc=$?; cat gpurun_out/tune_uw.log
timeout 600 python scripts/tune.py C5 'uw_bits=1' 'uw_bits=0' > gpurun_out/tune_uw5.log 2>&1; echo tune5 rc=$?; cat gpurun_out/tune_uw5.log
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:"k_tc_|k_uw_" --csv --log-file gpurun_out/uw_ncu.csv python scripts/run_tc.py --config C4 --reps 1 --what support > gpurun_out/uw_ncu.log 2>&1; echo ncu rc=$?
