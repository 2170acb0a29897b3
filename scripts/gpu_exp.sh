timeout 1500 python -m pytest tests -m gpu -x -q -p no:warnings -k "c4_full or analysis" 2>&1 | tail -2
