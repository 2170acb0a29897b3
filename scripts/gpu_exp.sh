GC_PEEL_TRACE=2 timeout 1500 python scripts/run_decomp.py --config C5 > gpurun_out/trace_c5r.log 2>&1; tail -1 gpurun_out/trace_c5r.log
