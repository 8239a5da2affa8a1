#!/bin/bash
# c5 final LAP and the tie-heavy n = 7500 case under the stall / tail knobs
cd $GRAFT_REPO_ROOT
for cfg in "GOAT_LAP_STALL=0" "GOAT_LAP_STALL=16" "GOAT_LAP_STALL=64" "GOAT_LAP_STALL=256"; do
  echo "== tied7500 $cfg"
  env $cfg GOAT_LAP_VERBOSE=1 timeout 600 python -m pytest tests/test_lap_auction_gpu.py -q -x -p no:cacheprovider -k "large_order and tied" -s 2>&1 | grep "lap n=\|passed\|failed" | cut -c1-300
done
for cfg in "GOAT_LAP_STALL=16" "GOAT_LAP_STALL=64" "GOAT_LAP_STALL=256" "GOAT_LAP_STALL=64 GOAT_LAP_TAIL=8192" "GOAT_LAP_STALL=16 GOAT_LAP_TAIL=0"; do
  echo "== c5 $cfg"
  env $cfg GOAT_LAP_VERBOSE=1 timeout 600 python scripts/run_c5.py 5 40000 fp32 csr 2>&1 | grep -v "^$" | cut -c1-420 | tail -4
done
