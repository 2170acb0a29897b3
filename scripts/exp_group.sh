python -m pytest tests/test_parity_gpu.py -q -x -m gpu -k "grouped or fuzz or golden or c3 or compaction or c1 or c5 or king or partition" 2>&1 | tail -3
for cfg in C3 C4 C5; do
  timeout 300 python scripts/run_decomp.py --config $cfg 2>&1 | grep -E "decomposition"
done
