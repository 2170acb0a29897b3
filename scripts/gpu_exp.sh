for L in sw9 sw11; do echo $L; GC_LIB_PATH=exp/libgc_$L.so timeout 600 python scripts/tune.py C4 "long_seg=48" 2>&1 | tail -1; done
