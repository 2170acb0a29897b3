python -m pytest tests/test_parity_gpu.py -q -x -m gpu -k "c1 or c3 or fuzz or compaction or grouped or golden or partition or king" 2>&1 | tail -2
for lib in build_var/prev/libgc.so paper_1708_06866_b200/libgc.so build_var/m0/libgc.so build_var/m8/libgc.so; do
echo $lib
for cfg in C4 C5; do GC_LIB_PATH=$lib timeout 300 python scripts/run_decomp.py --config $cfg --ks 4,6 2>&1 | grep -E "decomposition|ktruss" | cut -c1-150; done
done
