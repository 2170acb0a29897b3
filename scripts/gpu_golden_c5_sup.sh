# C5 golden, supports only (O-3 from the box's cache of the last call, T = sum / 3): gpurun_out/c5_expected.json
mkdir -p gpurun_out
ls -la /tmp/golden_cache_c5 > gpurun_out/golden_c5_sup.log 2>&1
GOLDEN_CACHE=/tmp/golden_cache_c5 timeout 3000 python scripts/make_golden.py --support-only C5 >> gpurun_out/golden_c5_sup.log 2>&1
echo "rc=$?" >> gpurun_out/golden_c5_sup.log
cp tests/golden/c5_expected.json gpurun_out/ 2>/dev/null
tail -4 gpurun_out/golden_c5_sup.log
