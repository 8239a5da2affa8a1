#!/bin/bash
# table-based fp64 exp: fp64 parity + per-sweep times
cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests/test_parity_gpu.py tests/test_full_configs_gpu.py tests/test_lot_large_gpu.py tests/test_sharded_gpu.py tests/test_configs_gpu.py -q -p no:cacheprovider > gpurun_out/r2m_tests.log 2>&1
tail -5 gpurun_out/r2m_tests.log
for n in 100 1000 5000 20000 40000; do python scripts/prof_sweep.py $n fp64 20; done
python scripts/run_c5.py 5 40000 fp32 csr 2>&1 | tail -1 | cut -c1-400
