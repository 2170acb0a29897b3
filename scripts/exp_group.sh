for o in "2=32768" "2=65536" "2=131072" "2=16384" "5=32" "5=64" "5=96"; do
echo $o; python scripts/run_tc.py --config C4 --reps 3 --what tc,support --opt $o | tail -1 | cut -c1-130
done
