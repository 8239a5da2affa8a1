#!/bin/bash
# fp64 sweep at n = 40000 / 20000: planner knobs
cd $GRAFT_REPO_ROOT
for cfg in "GOAT_SK_VERBOSE=1" "GOAT_SK_TMA=0" "GOAT_SK_STAGES=3" "GOAT_SK_STAGES=4" "GOAT_SK_STAGES=6" "GOAT_SK_MAXCH=4" "GOAT_SK_MAXCH=6" "GOAT_SK_RES=0"; do
  echo "== $cfg"; env $cfg python scripts/prof_sweep.py 40000 fp64 6 2>&1 | tail -2
done
for cfg in "GOAT_SK_VERBOSE=1" "GOAT_SK_TMA=0" "GOAT_SK_MAXCH=4"; do
  echo "== n=20000 $cfg"; env $cfg python scripts/prof_sweep.py 20000 fp64 10 2>&1 | tail -1
done
