#!/bin/bash
# round 2, first GPU pass: GPU suite (incl. full-size c3/c4), fp32 status, new c5 bench
cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2a_smi.txt 2>&1
timeout 900 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/r2a_tests.log 2>&1
timeout 600 python scripts/fp32_status.py fp32,fp64 > gpurun_out/r2a_fp32.jsonl 2> gpurun_out/r2a_fp32.err
timeout 1200 python bench.py --steps 2 --warmup 3 > gpurun_out/r2a_bench.json 2> gpurun_out/r2a_bench.err
tail -3 gpurun_out/r2a_tests.log
