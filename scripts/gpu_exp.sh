timeout 1500 python -m pytest tests -m gpu -x -q -p no:warnings -k "fuzz" 2>&1 | tail -15
