mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_parity_gpu.py -x -q -p no:warnings -k "loopback or partitioned or nccl or fuzz or analysis_one_pass" > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest_gpu.log
timeout 1200 python scripts/loopback_scaling.py C4 --parts 0,2,4,8 > gpurun_out/loopback_c4.log 2>&1; echo loop rc=$?; cat gpurun_out/loopback_c4.log
