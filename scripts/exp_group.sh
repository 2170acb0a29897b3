python scripts/run_tc.py --config C4 --reps 3 --what tc | tail -2 | cut -c1-100
python -m pytest tests/test_parity_gpu.py -q -x -m gpu -k "c1 or c3 or c4 or golden or empty or loops or duplicates or staged" 2>&1 | tail -1
