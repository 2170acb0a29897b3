timeout 1500 python -m pytest tests -m gpu -x -q -p no:warnings -k "grouped or peel or decomposition or golden or c1 or c3" 2>&1 | tail -2
for C in C3 C4 C5 K13; do for G in 0 16384; do echo "$C group=$G"; timeout 900 python scripts/run_decomp.py --config $C --ks 6 --group $G 2>&1 | tail -2; done; done
