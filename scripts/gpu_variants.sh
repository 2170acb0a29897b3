mkdir -p gpurun_out
timeout 600 python scripts/tune.py C4 '' '' '' > gpurun_out/variants.log 2>&1
timeout 600 python scripts/tune.py C5 '' >> gpurun_out/variants.log 2>&1
timeout 900 python -m pytest tests/test_parity_gpu.py -x -q -p no:warnings -k "forced or heavy or huge or task_chunk or fuzz or c4_full or large_clique or loopback" >> gpurun_out/variants.log 2>&1
cat gpurun_out/variants.log | tail -12
