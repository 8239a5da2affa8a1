#!/bin/bash
# single-CTA warm repairs: level-wise solver (cluster of one) vs the single-column solver, at c3 / c4 sizes
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_lap_auction_gpu.py tests/test_parity_gpu.py -q -x -p no:cacheprovider > gpurun_out/r2m_tests.log 2>&1
tail -3 gpurun_out/r2m_tests.log
for lv in 0 1; do
  echo "== GOAT_LAP_LEVELS=$lv"
  GOAT_LAP_LEVELS=$lv GOAT_LAP_VERBOSE=1 timeout 600 python scripts/fp32_status.py fp32 2>&1 >/dev/null | grep "lap n=" | cut -c1-260
done
