for lib in paper_1708_06866_b200/libgc.so build_var/v4/libgc.so build_var/v4w12/libgc.so; do
echo $lib
GC_LIB_PATH=$lib python scripts/run_tc.py --config C4 --reps 3 --what tc,support | tail -1 | cut -c1-130
done
