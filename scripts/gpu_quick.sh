timeout 600 python scripts/debug_support2.py 16
timeout 900 python -m pytest tests -m gpu -x -q -p no:warnings 2>&1 | tail -3
timeout 300 python scripts/run_tc.py --config C4 --reps 2 --what tc,support,ktruss 2>&1 | tail -2
