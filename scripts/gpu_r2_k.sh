#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_full_configs_gpu.py -q -p no:cacheprovider > gpurun_out/r2k_tests.log 2>&1
tail -5 gpurun_out/r2k_tests.log
bash scripts/conformance.sh > gpurun_out/r2k_conformance.log 2>&1
tail -6 gpurun_out/r2k_conformance.log
bash scripts/gpu_r2_lap.sh > gpurun_out/r2k_lap_scan.log 2>&1
cat gpurun_out/r2k_lap_scan.log
