python -m pytest tests/test_parity_gpu.py -q -x -m gpu -k "c3 or c4 or fuzz or golden or forced or heavy or huge or loopback" 2>&1 | tail -2
for i in 1 2; do
python scripts/run_tc.py --config C4 --reps 3 --what support | tail -1
GC_LIB_PATH=build_var/static/libgc.so python scripts/run_tc.py --config C4 --reps 3 --what support | tail -1
done
python scripts/run_tc.py --config C5 --reps 2 --what tc,support | tail -1
GC_LIB_PATH=build_var/static/libgc.so python scripts/run_tc.py --config C5 --reps 2 --what tc,support | tail -1
