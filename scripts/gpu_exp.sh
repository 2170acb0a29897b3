timeout 1500 python -m pytest tests -m gpu -x -q -p no:warnings 2>&1 | tail -2
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo bench rc=$?; tail -1 gpurun_out/bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); [print(k, d[k]) for k in ['value','ms_per_step','separate_calls','e2e','phase_ms','deeper']]"
