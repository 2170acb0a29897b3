set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
nproc
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
tail -5 gpurun_out/smoke.log
timeout 900 python -m pytest tests -m gpu -x -q -p no:warnings > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -30 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --config C3 --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/bench_c3.log 2>&1; echo bench3 rc=$?
tail -3 gpurun_out/bench_c3.log
timeout 900 python bench.py --steps 3 --warmup 2 > gpurun_out/bench_c4.log 2>&1; echo bench4 rc=$?
tail -3 gpurun_out/bench_c4.log
