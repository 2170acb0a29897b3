python scripts/run_tc.py --config C4 --reps 3 --what tc,support | tail -1 | cut -c1-130
python scripts/run_tc.py --config C5 --reps 2 --what tc,support | tail -1 | cut -c1-130
python -m pytest tests/test_parity_gpu.py -q -x -m gpu 2>&1 | tail -1
