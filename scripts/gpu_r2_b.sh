#!/bin/bash
# round 2: wide-row Sinkhorn kernels -- parity, then per-sweep scan
cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_wide_gpu.py tests/test_lot_large_gpu.py -q -x -p no:cacheprovider > gpurun_out/r2b_tests.log 2>&1
timeout 900 python scripts/sk_scan.py gpurun_out/r2b_scan.json \
  "16384,fp32,GOAT_SK_WIDE=0" "16384,fp32,GOAT_SK_VERBOSE=1" "16384,fp32,GOAT_SK_WIDE=4" \
  "20000,fp32,GOAT_SK_WIDE=0" "20000,fp32,GOAT_SK_VERBOSE=1" "20000,fp32,GOAT_SK_WIDE=4" \
  "32768,fp32,GOAT_SK_WIDE=0" "32768,fp32,GOAT_SK_VERBOSE=1" "32768,fp32,GOAT_SK_WIDE=4" \
  "40000,fp32,GOAT_SK_WIDE=0" "40000,fp32,GOAT_SK_VERBOSE=1" "40000,fp32,GOAT_SK_WIDE=4;GOAT_SK_STAGES=6" "40000,fp32,GOAT_SK_STAGES=6" "40000,fp32,GOAT_SK_STAGES=8" "40000,fp32,GOAT_SK_STAGES=10" \
  > gpurun_out/r2b_scan.log 2>&1
tail -3 gpurun_out/r2b_tests.log
cat gpurun_out/r2b_scan.log
