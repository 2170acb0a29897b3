mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:warnings 2>&1 | tail -3
timeout 600 python scripts/tune.py C4 "sup_uw=0" 2>&1 | tail -2
timeout 1500 python scripts/run_decomp.py --config C5 --tc 2 --no-decomp 2>&1 | tail -4
