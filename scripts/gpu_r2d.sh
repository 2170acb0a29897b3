mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -p no:warnings -k "not c4_full and not c5_full" > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -5 gpurun_out/pytest_gpu.log
timeout 1200 python scripts/loopback_scaling.py C4 --decomp > gpurun_out/loopback_c4.log 2>&1; echo loop rc=$?; cat gpurun_out/loopback_c4.log
