timeout 900 python scripts/stress_api.py 2>&1 | tail -3
