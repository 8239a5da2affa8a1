#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_sharded_gpu.py -q -p no:cacheprovider 2>&1 | tail -2
GOAT_SK_FP64_FINISH=0 python scripts/prof_shard_sweep.py 40000 100 fp32 2>&1 | tail -1
python scripts/prof_shard_sweep.py 40000 30 fp64 2>&1 | tail -1
GOAT_SK_FP64_FINISH=0 python scripts/prof_shard_sweep.py 5000 200 fp32 2>&1 | tail -1
