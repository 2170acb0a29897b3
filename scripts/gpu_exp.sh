mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q -p no:warnings -k "not c5" 2>&1 | tail -2
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench.log 2>&1; echo bench rc=$?; tail -1 gpurun_out/bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); [print(k, d[k]) for k in ['value','ms_per_step','roofline','roofline_tc','cpu_baseline','e2e','phase_ms']]"
timeout 600 python scripts/run_decomp.py --config C4 2>&1 | tail -1
