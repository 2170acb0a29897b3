for lib in paper_1708_06866_b200/libgc.so build_var/h20m3/libgc.so; do
echo $lib
GC_LIB_PATH=$lib python scripts/run_tc.py --config C5 --reps 2 --what tc | tail -1 | cut -c1-100
done
python -m pytest tests/test_parity_gpu.py -q -x -m gpu -k "huge or c5 or forced or large" 2>&1 | tail -1
