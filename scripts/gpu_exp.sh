for C in K13 C4 C2; do timeout 600 python scripts/tune.py $C "long_seg=48" 2>&1 | tail -1; done
timeout 900 python -m pytest tests -m gpu -x -q -p no:warnings -k "c1 or c2 or king or golden" 2>&1 | tail -1
