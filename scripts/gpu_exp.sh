timeout 1200 python -m pytest tests -m gpu -x -q -p no:warnings -k "forced or heavy or huge or chunk or c3 or c1 or golden or clique or loopback or c2 or king" 2>&1 | tail -2
for L in t16 t256; do echo $L; GC_LIB_PATH=exp/libgc_$L.so timeout 600 python scripts/tune.py C4 "overlap=1" 2>&1 | tail -1; done
echo t64; timeout 600 python scripts/tune.py C4 "overlap=1" 2>&1 | tail -1
timeout 600 python scripts/tune.py K13 "overlap=1" 2>&1 | tail -1
