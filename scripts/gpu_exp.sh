timeout 1500 python -m pytest tests -m gpu -x -q -p no:warnings -k "not c5" 2>&1 | tail -2
for C in C4 K13; do timeout 600 python scripts/run_tc.py --config $C --reps 3 --what tc 2>&1 | tail -1 | cut -c1-70; done
