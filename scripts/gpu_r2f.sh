mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_parity_gpu.py -x -q -p no:warnings -k "partitioned_build or loopback or nccl or partitioned_peeler" > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -5 gpurun_out/pytest_gpu.log
timeout 900 python scripts/build_ab.py C4 > gpurun_out/build_ab.log 2>&1; echo build_ab rc=$?; cat gpurun_out/build_ab.log
