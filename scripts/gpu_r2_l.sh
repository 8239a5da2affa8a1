#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests/test_lap_auction_gpu.py tests/test_configs_gpu.py -q -p no:cacheprovider -x > gpurun_out/r2l_tests.log 2>&1
tail -3 gpurun_out/r2l_tests.log
bash scripts/gpu_r2_lap.sh > gpurun_out/r2l_lap_scan.log 2>&1
cat gpurun_out/r2l_lap_scan.log
