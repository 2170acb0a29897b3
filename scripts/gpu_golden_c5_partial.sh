# C5 golden on the GPU box's host cores in one call, O-8 up to a deadline (O8_DEADLINE_S from the start of
# this script): O-3 supports, T = sum / 3, then O-8; if O-8 stops at the deadline the golden holds the exact
# trussness clipped at the last finished level (trussness_partial).  Then test_c5_full against it.
mkdir -p gpurun_out
L=gpurun_out/golden_c5.log
{ date; nproc; free -g | head -2; ls -la /tmp/golden_cache_c5 2>/dev/null; } > $L
GOLDEN_DEADLINE=$(( $(date +%s) + ${O8_DEADLINE_S:-5400} )) GOLDEN_CACHE=/tmp/golden_cache_c5 \
  python scripts/make_golden.py --ckpt /tmp/golden_cache_c5/o8.ckpt 0 C5 >> $L 2>&1
rc=$?
echo "make_golden rc=$rc $(date)" >> $L
if [ $rc = 0 ] || [ $rc = 3 ]; then
  cp tests/golden/c5_expected.json gpurun_out/
  timeout 1200 python -m pytest tests/test_parity_gpu.py -m gpu -q -p no:warnings -rxX -k "test_c5_full" \
    > gpurun_out/pytest_c5.log 2>&1
  echo "pytest c5 rc=$?" >> $L
  tail -4 gpurun_out/pytest_c5.log >> $L
fi
tail -12 $L
