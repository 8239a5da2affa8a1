#!/bin/bash
# thread-0 phase-cycle accounting of one fixed-shift sweep of the TM wide kernel at n = 40000
cd $GRAFT_REPO_ROOT
GOAT_SK_TRACE=5 GOAT_SK_TRACE_RAW=1 python scripts/prof_sweep.py 40000 fp32 8 > gpurun_out/r2e_trace.log 2>&1
GOAT_SK_TRACE=1 GOAT_SK_TRACE_RAW=1 python scripts/prof_sweep.py 40000 fp32 8 >> gpurun_out/r2e_trace.log 2>&1
cat gpurun_out/r2e_trace.log
