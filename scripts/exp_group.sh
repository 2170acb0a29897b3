python scripts/run_tc.py --config C4 --reps 3 --what tc,support | tail -2 | cut -c1-200
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_tf.csv -k regex:k_task_flags python scripts/run_tc.py --config C4 --reps 1 --what tc > /dev/null 2>&1; grep k_task_flags gpurun_out/launches_tf.csv | tail -1 | cut -c1-50,150-
python -m pytest tests/test_parity_gpu.py -q -x -m gpu -k "c3 or c4 or chunk or loopback or golden" 2>&1 | tail -1
