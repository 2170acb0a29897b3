mkdir -p gpurun_out
timeout 2400 python scripts/run_configs.py --configs C1,C2,C3,C4,C5 --oracle --out gpurun_out/configs > gpurun_out/configs.log 2>&1; echo configs rc=$?; tail -3 gpurun_out/configs.log | cut -c1-400; cat gpurun_out/configs/configs.md
