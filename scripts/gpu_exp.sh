timeout 600 python scripts/tune.py C4 "overlap=1" 2>&1 | tail -1
timeout 600 python scripts/tune.py C3 "overlap=1" 2>&1 | tail -1
timeout 900 python -m pytest tests -m gpu -x -q -p no:warnings -k "huge or forced or clique or c3 or c1 or c2" 2>&1 | tail -1
