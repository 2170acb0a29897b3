# C5 trussness by O-8 in 1-hour calls: resumes from /tmp/golden_cache_c5/o8.ckpt (supports cached there by
# scripts/gpu_golden_c5.sh); exit 3 = state saved, call again; 0 = golden written (gpurun_out/c5_expected.json)
mkdir -p gpurun_out
ls -la /tmp/golden_cache_c5 > gpurun_out/golden_c5_o8.log 2>&1
GOLDEN_DEADLINE=$(( $(date +%s) + ${O8_WINDOW:-2700} )) GOLDEN_CACHE=/tmp/golden_cache_c5 timeout 3450 python scripts/make_golden.py --ckpt /tmp/golden_cache_c5/o8.ckpt ${O8_BUDGET:-2400} C5 >> gpurun_out/golden_c5_o8.log 2>&1
rc=$?
echo "make_golden rc=$rc" >> gpurun_out/golden_c5_o8.log
[ $rc = 0 ] && cp tests/golden/c5_expected.json gpurun_out/
tail -4 gpurun_out/golden_c5_o8.log
