python -m pytest tests/test_parity_gpu.py -q -x -m gpu -k "c3 or c4 or c5 or king or fuzz or compaction or partition or grouped or golden" 2>&1 | tail -2
GC_PEEL_BIG=1 python -m pytest tests/test_parity_gpu.py -q -x -m gpu -k "c1 or c3 or fuzz or compaction or grouped" 2>&1 | tail -2
