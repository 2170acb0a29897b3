for lib in build_var/prev3/libgc.so paper_1708_06866_b200/libgc.so build_var/prev3/libgc.so paper_1708_06866_b200/libgc.so; do
echo $lib
GC_LIB_PATH=$lib python scripts/run_tc.py --config C4 --reps 3 --what support | tail -1 | cut -c1-130
done
GC_LIB_PATH=build_var/prev3/libgc.so python scripts/run_tc.py --config C5 --reps 2 --what support | tail -1 | cut -c1-130
python scripts/run_tc.py --config C5 --reps 2 --what support | tail -1 | cut -c1-130
python -m pytest tests/test_parity_gpu.py -q -x -m gpu -k "c3 or c4 or forced or heavy or huge or golden or fuzz or random" 2>&1 | tail -1
