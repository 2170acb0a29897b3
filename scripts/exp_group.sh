python -m pytest tests/test_parity_gpu.py -q -x -m gpu -k "staged or golden or errors or device" 2>&1 | tail -2
python bench.py --steps 5 --warmup 3 --no-extra --no-cpu-baseline > gpurun_out/bench_tmp.log 2>&1; echo rc=$?
