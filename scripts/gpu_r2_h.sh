#!/bin/bash
# fp64-finish check: parity tests, fp32 status vs the reference goldens, FAQ parity, wide tests, reference suite
cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests/test_parity_gpu.py tests/test_full_configs_gpu.py tests/test_wide_gpu.py tests/test_configs_gpu.py -q -p no:cacheprovider > gpurun_out/r2h_tests.log 2>&1
tail -25 gpurun_out/r2h_tests.log
timeout 600 python scripts/fp32_status.py fp32 > gpurun_out/r2h_fp32.jsonl 2> gpurun_out/r2h_fp32.err
bash scripts/conformance.sh > gpurun_out/r2h_conformance.log 2>&1
tail -30 gpurun_out/r2h_conformance.log
