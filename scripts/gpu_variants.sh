mkdir -p gpurun_out
for V in "" build_var/first32/libgc.so "" build_var/first32/libgc.so; do
  echo "== ${V:-default}"
  GC_LIB_PATH=$V timeout 600 python scripts/peel_ab.py C4 '' 2>&1 | tail -1
done > gpurun_out/variants.log 2>&1
for V in "" build_var/first32/libgc.so; do
  echo "== C5 ${V:-default}"
  GC_LIB_PATH=$V timeout 600 python scripts/peel_ab.py C5 '' 2>&1 | tail -1
done >> gpurun_out/variants.log 2>&1
GC_LIB_PATH=build_var/first32/libgc.so timeout 900 python -m pytest tests/test_parity_gpu.py -x -q -p no:warnings -k "c1_full or compaction or register_builds or partitioned_peeler or golden_examples or fuzz or c4_full or random_small or complete" >> gpurun_out/variants.log 2>&1
cat gpurun_out/variants.log | tail -14
