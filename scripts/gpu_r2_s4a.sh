# session check: smoke, every -m gpu test with durations, the bench line, then the bulk-prefetch A/B
mkdir -p gpurun_out
{ nproc; free -g | head -2; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader; } > gpurun_out/box.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?; tail -1 gpurun_out/smoke.log
timeout 2400 python -m pytest tests -m gpu -q -p no:warnings -rxX --durations=15 > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -25 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.log 2>&1; echo bench rc=$?; tail -1 gpurun_out/bench.log | cut -c1-400
bash scripts/gpu_pf_ab.sh
