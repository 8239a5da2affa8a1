#!/bin/bash
cd $GRAFT_REPO_ROOT
GOAT_LAP_VERBOSE=1 timeout 900 python -m pytest tests/test_lap_auction_gpu.py -q -x -p no:cacheprovider -k "12000" -s > gpurun_out/r2m_tests.log 2>&1
grep "lap \|passed\|failed\|Error" gpurun_out/r2m_tests.log | cut -c1-250
