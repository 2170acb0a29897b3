python -m pytest tests/test_parity_gpu.py -q -x -m gpu -k "c1 or c3 or compaction or fuzz or golden or register or partition or grouped" 2>&1 | tail -1
for cfg in C4 C5; do timeout 300 python scripts/run_decomp.py --config $cfg --ks 4,5,6 2>&1 | grep -E "decomposition|ktruss" | cut -c1-170; done
