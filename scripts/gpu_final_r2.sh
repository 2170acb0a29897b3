# round-2 final check: smoke, every -m gpu test (C5 last), the C4 bench line, the per-config report
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?; tail -1 gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -q -p no:warnings -rxX > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -6 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.log 2>&1; echo bench rc=$?; tail -1 gpurun_out/bench.log | cut -c1-300
[ "${CONFIGS:-1}" = 1 ] && { timeout 1200 python scripts/run_configs.py --oracle > gpurun_out/configs.log 2>&1; echo configs rc=$?; }
cp profiles/round2/configs.md profiles/round2/configs.jsonl gpurun_out/ 2>/dev/null
true
