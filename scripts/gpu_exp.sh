for K in 96 128 192 384; do echo "kD1=$K"; GC_LIB_PATH=exp/libgc_k$K.so timeout 600 python scripts/tune.py C4 "overlap=1" 2>&1 | tail -1; done
echo "kD1=256"; timeout 600 python scripts/tune.py C4 "overlap=1" 2>&1 | tail -1
