python -m pytest tests/test_parity_gpu.py -q -x -m gpu -k "async or staged or golden or fused or analysis" 2>&1 | tail -2
python bench.py --steps 5 --warmup 3 --no-extra --no-cpu-baseline > gpurun_out/bench_tmp.log 2>&1; echo rc=$?
