for L in s12_4 s16_3 s10_4; do echo $L; GC_LIB_PATH=exp/libgc_$L.so timeout 600 python scripts/tune.py C4 "overlap=1" 2>&1 | tail -1; done
