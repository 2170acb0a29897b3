for lib in paper_1708_06866_b200/libgc.so build_var/dw8/libgc.so build_var/dw32/libgc.so; do
echo $lib
GC_LIB_PATH=$lib python scripts/run_tc.py --config C4 --reps 3 --what tc,support | tail -1 | cut -c1-130
GC_LIB_PATH=$lib python scripts/run_tc.py --config C5 --reps 2 --what tc,support | tail -1 | cut -c1-130
done
GC_LIB_PATH=build_var/dw8/libgc.so python -m pytest tests/test_parity_gpu.py -q -x -m gpu -k "c3 or c4 or forced or heavy or huge or golden or loopback" 2>&1 | tail -1
