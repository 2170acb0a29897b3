timeout 1500 python -m pytest tests -m gpu -x -q -p no:warnings -k "c1 or c2 or c3 or golden or king or random or degenerate or empty or self or single" 2>&1 | tail -1
for C in C4 K13 C5; do timeout 600 python scripts/run_tc.py --config $C --reps 3 --what tc 2>&1 | tail -1 | cut -c1-60; done
