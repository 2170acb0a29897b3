python -m pytest tests/test_parity_gpu.py -q -x -m gpu 2>&1 | tail -1
for cfg in C3 C4 C5 K13; do timeout 300 python scripts/run_decomp.py --config $cfg --ks 4,5,6 2>&1 | grep -E "decomposition|ktruss" | cut -c1-150; done
