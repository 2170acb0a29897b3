mkdir -p gpurun_out
timeout 900 python scripts/peel_ab.py C4 'sort_front=0' 'sort_front=1000000' 'sort_front=100000' 'sort_front=10000' 'sort_front=0' > gpurun_out/peel_ab.log 2>&1; echo ab rc=$?; cat gpurun_out/peel_ab.log
