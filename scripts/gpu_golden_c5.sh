# C5 golden on the GPU box's host cores (oracle only; the GPU is not used): O-3 supports, T = sum / 3,
# O-8 trussness -> gpurun_out/c5_expected.json (progress in gpurun_out/golden_c5.log)
mkdir -p gpurun_out
{ nproc; free -g | head -2; } > gpurun_out/golden_c5.log
GOLDEN_CACHE=/tmp/golden_cache_c5 python scripts/make_golden.py C5 >> gpurun_out/golden_c5.log 2>&1
echo "make_golden rc=$?" >> gpurun_out/golden_c5.log
cp tests/golden/c5_expected.json gpurun_out/ 2>/dev/null
tail -3 gpurun_out/golden_c5.log
