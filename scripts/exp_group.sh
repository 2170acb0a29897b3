for lib in paper_1708_06866_b200/libgc.so build_var/x3/libgc.so; do
echo $lib
for cfg in C4 C5 K13; do GC_LIB_PATH=$lib timeout 300 python scripts/run_decomp.py --config $cfg --ks 5,6 2>&1 | grep -E "decomposition|ktruss" | cut -c1-150; done
done
