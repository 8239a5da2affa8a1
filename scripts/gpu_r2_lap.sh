#!/bin/bash
# c5 final LAP: phase split
cd $GRAFT_REPO_ROOT
for cfg in "GOAT_LAP_TAIL=2048"; do
  echo "== $cfg"
  env $cfg GOAT_LAP_VERBOSE=1 timeout 600 python scripts/run_c5.py 5 40000 fp32 csr 2>&1 | grep -v "^$" | cut -c1-420 | tail -12
done
