timeout 900 python -m pytest tests -m gpu -x -q -p no:warnings -k "peel or decomposition or fuzz or golden or c1 or c3 or loopback or analysis" 2>&1 | tail -1
for C in C3 C4 C5 K13; do timeout 900 python scripts/run_decomp.py --config $C --ks 6 2>&1 | tail -2; done
