for M in 4 16 64; do echo "min=$M"; GC_LIB_PATH=exp/libgc_g$M.so timeout 900 python scripts/run_decomp.py --config C4 --ks 8 2>&1 | tail -2; done
echo "group=0"; timeout 900 python scripts/run_decomp.py --config C4 --ks 8 --group 0 2>&1 | tail -2
