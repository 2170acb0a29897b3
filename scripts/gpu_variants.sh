mkdir -p gpurun_out
for V in "" build_var/pair/libgc.so "" build_var/pair/libgc.so; do
  echo "== ${V:-default}"
  GC_LIB_PATH=$V timeout 600 python scripts/tune.py C4 '' 2>&1 | tail -1
done > gpurun_out/variants.log 2>&1
for V in "" build_var/pair/libgc.so; do
  echo "== C5 ${V:-default}"
  GC_LIB_PATH=$V timeout 600 python scripts/tune.py C5 '' 2>&1 | tail -1
done >> gpurun_out/variants.log 2>&1
GC_LIB_PATH=build_var/pair/libgc.so timeout 900 python -m pytest tests/test_parity_gpu.py -x -q -p no:warnings -k "forced or heavy or huge or task_chunk or fuzz or c4_full or large_clique or loopback or c1_full" >> gpurun_out/variants.log 2>&1
cat gpurun_out/variants.log | tail -14
