mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:warnings -k "not c5 and not c4" 2>&1 | tail -2
timeout 600 python scripts/tune.py C4 "sup_uw=0" 2>&1 | tail -1
timeout 600 python scripts/tune.py C3 "sup_uw=0" 2>&1 | tail -1
