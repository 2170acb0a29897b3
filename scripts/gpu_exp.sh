timeout 1200 python -m pytest tests -m gpu -x -q -p no:warnings -k "not c5 and not K13" 2>&1 | tail -2
timeout 600 python scripts/tune.py C4 "sup_skip=0" 2>&1 | tail -1
