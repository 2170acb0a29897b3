timeout 1200 python -m pytest tests -m gpu -x -q -p no:warnings -k "forced or heavy or huge or chunk or c3 or c1 or golden or clique" 2>&1 | tail -2
timeout 600 python scripts/tune.py C4 "sup_skip=0" "sup_skip=2" 2>&1 | tail -2
