timeout 900 python -m pytest tests -m gpu -x -q -p no:warnings -k "peel or decomposition or fuzz or c3" 2>&1 | tail -1
for L in w0 w64 w1024; do echo $L; for C in C4 C5; do GC_LIB_PATH=exp/libgc_$L.so timeout 900 python scripts/run_decomp.py --config $C --ks 6 2>&1 | tail -2; done; done
echo w256; for C in C4 C5; do timeout 900 python scripts/run_decomp.py --config $C --ks 6 2>&1 | tail -2; done
