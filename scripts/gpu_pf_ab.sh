# A/B of the TMA bulk L2 prefetch variants (GC_BULK_PF in the intersection kernels, GC_PEEL_PF in the
# peeler) against the in-tree build: parity of each variant, then C4 / C5 pass times -> gpurun_out/pf_ab.log
# (variants built by scripts/build_variant.sh pf1 -DGC_BULK_PF=1 / pf3 -DGC_BULK_PF=3 / pf5 -DGC_BULK_PF=5 / ppf -DGC_PEEL_PF=1)
mkdir -p gpurun_out
L=gpurun_out/pf_ab.log
: > $L
lib() { [ "$1" = default ] && echo "" || echo "build_var/$1/libgc.so"; }
for v in pf1 pf3 pf5; do
  echo "== parity $v" >> $L
  GC_LIB_PATH=$(lib $v) timeout 600 python -m pytest tests/test_parity_gpu.py -m gpu -q -x -p no:warnings \
    -k "forced or heavy or huge or chunk or c3_full" >> $L 2>&1; echo "rc=$?" >> $L
done
echo "== parity ppf" >> $L
GC_LIB_PATH=$(lib ppf) timeout 600 python -m pytest tests/test_parity_gpu.py -m gpu -q -x -p no:warnings \
  -k "ktruss or decomposition or c3_full or compaction" >> $L 2>&1; echo "rc=$?" >> $L
for r in 1 2; do
  for v in default pf1 pf3 pf5; do
    echo "== C4 tc/support $v (rep $r)" >> $L
    GC_LIB_PATH=$(lib $v) timeout 300 python scripts/tune.py C4 '' >> $L 2>&1
  done
done
for v in default ppf default ppf; do
  echo "== C4 peel $v" >> $L
  GC_LIB_PATH=$(lib $v) timeout 300 python scripts/peel_ab.py C4 '' >> $L 2>&1
done
for v in default pf1; do
  echo "== C5 tc/support $v" >> $L
  GC_LIB_PATH=$(lib $v) timeout 400 python scripts/tune.py C5 '' >> $L 2>&1
done
grep -E "^==|rc=|passed|failed|tc .* ms|peel" $L | tail -60
