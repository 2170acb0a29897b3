mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:warnings 2>&1 | tail -3
for cf in 0 2; do timeout 300 python scripts/run_decomp.py --config C3 --compact $cf 2>&1 | tail -1; done
for cf in 0 2; do timeout 600 python scripts/run_decomp.py --config C4 --compact $cf 2>&1 | tail -1; done
timeout 1500 python scripts/run_decomp.py --config C5 2>&1 | tail -1
