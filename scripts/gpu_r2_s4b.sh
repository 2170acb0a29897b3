# session check 2: the C3 / C5 tests with the trussness property checks, the round-2 profile set
# (scripts/gpu_profile_r2.sh), the per-config report (scripts/run_configs.py --oracle)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_parity_gpu.py -m gpu -q -p no:warnings -rxX --durations=5 \
  -k "c3_full or c5_full" > gpurun_out/pytest_props.log 2>&1; echo pytest rc=$?; tail -12 gpurun_out/pytest_props.log
bash scripts/gpu_profile_r2.sh
timeout 1500 python scripts/run_configs.py --oracle > gpurun_out/configs.log 2>&1; echo configs rc=$?
cp profiles/round2/configs.md profiles/round2/configs.jsonl gpurun_out/ 2>/dev/null
tail -5 gpurun_out/configs.log
