mkdir -p gpurun_out
cat > /tmp/b1.py <<'PY'
import os, sys
sys.path.insert(0, os.getcwd())
import torch, gen
from paper_1708_06866_b200 import gc
u, v = gen.CONFIGS["C4"].generate()
ctx = gc.Context(0, torch.cuda.current_stream())
ctx.load_edges(torch.from_numpy(u).cuda(), torch.from_numpy(v).cuda())
ctx.set_option(gc.GC_OPT_BUILD, int(sys.argv[1]))
ctx.build_csr()
print(ctx.stats()["build_ms"])
PY
for M in 1 0; do
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/build_ncu_$M.csv python /tmp/b1.py $M > gpurun_out/build_ncu_$M.log 2>&1; echo ncu $M rc=$?
done
