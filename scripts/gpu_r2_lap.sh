#!/bin/bash
# c5 final LAP: phase split; 8- vs 16-CTA cluster repair
cd $GRAFT_REPO_ROOT
for cfg in "GOAT_LAP_CL=16" "GOAT_LAP_CL=8"; do
  echo "== $cfg"
  env $cfg GOAT_LAP_VERBOSE=1 timeout 600 python scripts/run_c5.py 5 40000 fp32 csr 2>&1 | grep "repair\|auction kernel\|wall_s" | cut -c1-300
done
