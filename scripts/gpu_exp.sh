for L in k64 k96 k192; do echo $L; GC_LIB_PATH=exp/libgc_$L.so timeout 600 python scripts/tune.py C4 "long_seg=48" 2>&1 | tail -1; done
echo k128; timeout 600 python scripts/tune.py C4 "long_seg=48" 2>&1 | tail -1
