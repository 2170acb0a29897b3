# support-pass traffic by credit role (GC_OPT_SUP_SKIP, diagnostics): times and ncu DRAM bytes per kernel
mkdir -p gpurun_out
export GC_DIAG=1
timeout 600 python scripts/tune.py C4 'sup_skip=0' 'sup_skip=1' 'sup_skip=2' 'sup_skip=4' 'sup_skip=7' 'sup_skip=0' > gpurun_out/attrib_tune.log 2>&1; echo tune rc=$?; cat gpurun_out/attrib_tune.log
for S in 0 1 2 4 7; do
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum \
  --clock-control none -k regex:k_tc_ --csv --log-file gpurun_out/attrib_ncu_$S.csv \
  python scripts/run_tc.py --config C4 --reps 1 --what support --opt 7=$S > gpurun_out/attrib_ncu_$S.log 2>&1; echo ncu $S rc=$?
done
