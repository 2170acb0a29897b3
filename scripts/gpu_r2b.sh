mkdir -p gpurun_out
timeout 600 python scripts/build_ab.py C4 > gpurun_out/build_ab.log 2>&1; echo build_ab rc=$?; cat gpurun_out/build_ab.log
timeout 600 python scripts/build_ab.py C5 >> gpurun_out/build_ab.log 2>&1; echo build_ab5 rc=$?; tail -4 gpurun_out/build_ab.log
timeout 1500 python -m pytest tests -m gpu -x -q -p no:warnings -k "not c4_full and not c5_full" > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -5 gpurun_out/pytest_gpu.log
