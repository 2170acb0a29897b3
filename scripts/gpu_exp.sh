mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:warnings -k "forced or heavy or huge or chunk or c3 or loopback or c1 or golden" 2>&1 | tail -2
timeout 600 python scripts/tune.py C4 "sup_skip=0" "sup_skip=7" 2>&1 | tail -2
timeout 600 python scripts/tune.py C3 "sup_skip=0" 2>&1 | tail -1
