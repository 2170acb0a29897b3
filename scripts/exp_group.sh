for o in "13=1" "13=0" "13=1" "13=0"; do echo $o; python scripts/run_tc.py --config C4 --reps 3 --what tc,support --opt $o | tail -1 | cut -c1-120; done
