mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -p no:warnings --durations=8 2>&1 | tail -14
timeout 300 python scripts/run_decomp.py --config C4 2>&1 | tail -1
