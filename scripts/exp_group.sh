for lib in build_var/g64/libgc.so paper_1708_06866_b200/libgc.so; do
echo $lib
GC_LIB_PATH=$lib timeout 300 python scripts/run_decomp.py --config C4 2>&1 | grep decomposition | cut -c1-160
GC_LIB_PATH=$lib python scripts/run_tc.py --config C4 --reps 3 --what analysis | tail -1 | cut -c1-110
done
