for v in 5 10 20; do echo compact $v; for cfg in C4 C5; do timeout 300 python scripts/run_decomp.py --config $cfg --compact $v 2>&1 | grep decomposition | cut -c1-170; done; done
