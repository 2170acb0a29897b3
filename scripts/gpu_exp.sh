for G in 4 8 16; do echo G=$G; for C in C4 K13; do GC_LIB_PATH=exp/libgc_g$G.so timeout 900 python scripts/run_decomp.py --config $C 2>&1 | tail -1; done; done
