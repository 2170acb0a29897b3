timeout 1500 python -m pytest tests -m gpu -x -q -p no:warnings -k "not c5 and not c4" 2>&1 | tail -1
timeout 600 python scripts/tune.py C4 "long_seg=48" 2>&1 | tail -1
