timeout 600 python scripts/tune.py C5 "overlap=1" 2>&1 | tail -1
timeout 900 python -m pytest tests -m gpu -x -q -p no:warnings -k "huge or forced or clique or c3" 2>&1 | tail -1
