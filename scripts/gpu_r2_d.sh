#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_wide_gpu.py tests/test_lot_large_gpu.py -q -x -p no:cacheprovider > gpurun_out/r2d_tests.log 2>&1
timeout 900 python scripts/sk_scan.py gpurun_out/r2d_scan.json \
  "40000,fp32,GOAT_SK_VERBOSE=1" "40000,fp32,GOAT_SK_DBG=64" "40000,fp32,GOAT_SK_STAGES=3" \
  "32768,fp32,GOAT_SK_VERBOSE=1" "32768,fp32,GOAT_SK_WIDE=0" "25000,fp32,GOAT_SK_VERBOSE=1" "25000,fp32,GOAT_SK_WIDE=0" \
  "20000,fp32,GOAT_SK_VERBOSE=1" "20000,fp32,GOAT_SK_WIDE=0" "16384,fp32,GOAT_SK_VERBOSE=1" "16384,fp32,GOAT_SK_WIDE=0" \
  "13000,fp32,GOAT_SK_VERBOSE=1" "13000,fp32,GOAT_SK_WIDE=0" \
  > gpurun_out/r2d_scan.log 2>&1
tail -2 gpurun_out/r2d_tests.log; cat gpurun_out/r2d_scan.log
