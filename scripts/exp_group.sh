python -m pytest tests/test_parity_gpu.py -q -x -m gpu 2>&1 | tail -1
python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_tmp.log 2>&1; echo rc=$?
