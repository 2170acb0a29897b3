timeout 1200 python -m pytest tests -m gpu -x -q -p no:warnings -k "forced or heavy or huge or chunk or c3 or c1 or golden or clique or loopback or device" 2>&1 | tail -2
timeout 600 python scripts/tune.py C4 "overlap=1" "overlap=0" "overlap=1" 2>&1 | tail -3
timeout 600 python scripts/tune.py C5 "overlap=1" "overlap=0" 2>&1 | tail -2
