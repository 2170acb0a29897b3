mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:warnings -k "loopback or partitioned or golden" 2>&1 | tail -3
timeout 300 python scripts/run_decomp.py --config C1 2>&1 | tail -3
timeout 300 python scripts/run_decomp.py --config C1 --part 1 2>&1 | tail -1
timeout 300 python scripts/run_decomp.py --config C3 --ks 3,4,5,6 2>&1 | tail -6
timeout 300 python scripts/run_decomp.py --config C3 --ks 3,4,5,6 --part 1 2>&1 | tail -6
timeout 600 python scripts/run_decomp.py --config C4 --ks 3,8 2>&1 | tail -4
