for lib in paper_1708_06866_b200/libgc.so build_var/wm8/libgc.so paper_1708_06866_b200/libgc.so build_var/wm8/libgc.so; do
echo $lib
GC_LIB_PATH=$lib python scripts/run_tc.py --config C4 --reps 3 --what tc,support --opt 13=0 | tail -1 | cut -c1-130
GC_LIB_PATH=$lib python scripts/run_tc.py --config C4 --reps 3 --what tc,support | tail -1 | cut -c1-130
GC_LIB_PATH=$lib python scripts/run_tc.py --config C5 --reps 2 --what tc,support | tail -1 | cut -c1-130
done
