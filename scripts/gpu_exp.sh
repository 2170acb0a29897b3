timeout 1500 python -m pytest tests -m gpu -x -q -p no:warnings -k "analysis or golden or c1 or c3 or king" 2>&1 | tail -2
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench.log 2>&1; echo bench rc=$?; tail -1 gpurun_out/bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); [print(k, d[k]) for k in ['value','ms_per_step','phase_ms']]"
