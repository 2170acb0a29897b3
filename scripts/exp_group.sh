python -m pytest tests/test_parity_gpu.py -q -x -m gpu -k "c3 or c4 or fuzz or golden or rmat or c1 or analysis" 2>&1 | tail -3
python scripts/run_tc.py --config C4 --reps 3 --what analysis
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python scripts/run_tc.py --config C4 --reps 1 --what analysis > /dev/null 2>&1
python bench.py --steps 5 --warmup 3 --no-extra --no-cpu-baseline > gpurun_out/bench_tmp.log 2>&1
