timeout 1200 python -m pytest tests -m gpu -x -q -p no:warnings -k "not c5 and not c4" 2>&1 | tail -2
for C in C3 C4 C4 C5; do timeout 600 python scripts/run_decomp.py --config $C --ks 3,8 2>&1 | tail -3; done
