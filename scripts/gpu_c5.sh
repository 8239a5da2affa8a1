GOAT_LAP_VERBOSE=1 timeout 1500 python scripts/run_c5.py 3 2>&1 | tail -4 | cut -c1-700
