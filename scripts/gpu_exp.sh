timeout 1500 python -m pytest tests -m gpu -x -q -p no:warnings 2>&1 | tail -2
