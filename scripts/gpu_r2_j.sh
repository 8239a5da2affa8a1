#!/bin/bash
# full GPU suite + sharded bench at world 1 (refine) + bench + reference CLI tests
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider --durations=8 > gpurun_out/r2j_tests.log 2>&1
tail -14 gpurun_out/r2j_tests.log
bash scripts/conformance.sh > gpurun_out/r2j_conformance.log 2>&1
tail -6 gpurun_out/r2j_conformance.log
GOAT_BENCH_SHARDED=1 timeout 1500 python bench.py --steps 1 --warmup 3 > gpurun_out/r2j_bench_sharded_w1.json 2> gpurun_out/r2j_bench_sharded_w1.err; echo "sharded rc=$?"
cut -c1-900 gpurun_out/r2j_bench_sharded_w1.json
timeout 1500 python bench.py --steps 2 --warmup 3 > gpurun_out/r2j_bench.json 2> gpurun_out/r2j_bench.err; echo "bench rc=$?"
cut -c1-1500 gpurun_out/r2j_bench.json
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r2j_bench_ref.json 2> gpurun_out/r2j_bench_ref.err; echo "ref rc=$?"
