timeout 600 python scripts/tune.py C4 "long_seg=48" 2>&1 | tail -1
timeout 900 python -m pytest tests -m gpu -x -q -p no:warnings -k "forced or heavy or c3 or c1 or fuzz" 2>&1 | tail -1
