# full-size golden parity (C3, C4, and C5 once its golden exists)
mkdir -p gpurun_out
timeout 2400 python -m pytest tests/test_parity_gpu.py -x -q -p no:warnings -k "c3_full or c4_full or c5_full" > gpurun_out/pytest_golden.log 2>&1; echo pytest rc=$?; tail -15 gpurun_out/pytest_golden.log
