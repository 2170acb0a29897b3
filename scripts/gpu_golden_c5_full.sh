# C5 golden in one call on the GPU box's host cores (oracle only; the GPU is used only afterwards, by
# test_c5_full): O-3 supports, T = sum / 3, O-8 trussness up to a wall-clock deadline (O8_DEADLINE_S from
# the start), then the GPU parity test against the golden just written -> gpurun_out/c5_expected.json
mkdir -p gpurun_out
L=gpurun_out/golden_c5_full.log
{ date; nproc; free -g | head -2; } > $L
GOLDEN_DEADLINE=$(( $(date +%s) + ${O8_DEADLINE_S:-8100} )) GOLDEN_CACHE=/tmp/golden_cache_c5 \
  python scripts/make_golden.py --ckpt /tmp/golden_cache_c5/o8.ckpt 0 C5 >> $L 2>&1
rc=$?
echo "make_golden rc=$rc $(date)" >> $L
if [ $rc = 0 ]; then
  cp tests/golden/c5_expected.json gpurun_out/
  timeout 900 python -m pytest tests/test_parity_gpu.py -m gpu -q -p no:warnings -rxX -k "test_c5_full" \
    > gpurun_out/pytest_c5.log 2>&1
  echo "pytest c5 rc=$?" >> $L
  tail -3 gpurun_out/pytest_c5.log >> $L
fi
tail -8 $L
