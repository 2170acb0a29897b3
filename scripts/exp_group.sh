for lib in build_var/old/libgc.so paper_1708_06866_b200/libgc.so build_var/static/libgc.so; do
echo $lib
GC_LIB_PATH=$lib python scripts/run_tc.py --config C4 --reps 3 --what analysis | cut -c1-120
GC_LIB_PATH=$lib python scripts/run_tc.py --config C5 --reps 2 --what tc,support | cut -c1-120
done
