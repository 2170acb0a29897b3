mkdir -p gpurun_out
for V in build_var/base/libgc.so "" build_var/base/libgc.so ""; do
  echo "== ${V:-new}"
  GC_LIB_PATH=$V timeout 600 python scripts/peel_ab.py C4 '' 2>&1 | tail -1
done > gpurun_out/variants.log 2>&1
for V in build_var/base/libgc.so ""; do
  echo "== C5 ${V:-new}"
  GC_LIB_PATH=$V timeout 600 python scripts/peel_ab.py C5 '' 2>&1 | tail -1
done >> gpurun_out/variants.log 2>&1
timeout 900 python -m pytest tests/test_parity_gpu.py -x -q -p no:warnings -k "c1_full or compaction or register_builds or golden_examples or fuzz or c4_full or c3_full or random_small or complete or work_stats" >> gpurun_out/variants.log 2>&1
cat gpurun_out/variants.log | tail -14
