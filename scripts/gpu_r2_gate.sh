#!/bin/bash
# round 2 gate: GPU suite, reference suite, fp32 status, c5 bench (plain, both arms), ncu launch list of the same command
cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2g_smi.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2g_smoke.log 2>&1; echo "smoke rc=$?"
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider --durations=10 > gpurun_out/r2g_tests.log 2>&1
tail -4 gpurun_out/r2g_tests.log
bash scripts/conformance.sh > gpurun_out/r2g_conformance.log 2>&1
tail -7 gpurun_out/r2g_conformance.log
timeout 600 python scripts/fp32_status.py fp32 > gpurun_out/r2g_fp32.jsonl 2> gpurun_out/r2g_fp32.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r2g_bench_ref.json 2> gpurun_out/r2g_bench_ref.err; echo "ref rc=$?"
timeout 1500 python bench.py --steps 3 --warmup 3 > gpurun_out/r2g_bench.json 2> gpurun_out/r2g_bench.err; echo "bench rc=$?"
GOAT_BENCH_SECONDARY=0 timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/r2g_launches.csv python bench.py --steps 1 --warmup 3 > gpurun_out/r2g_ncu_bench.log 2>&1; echo "ncu list rc=$?"
GOAT_BENCH_SHARDED=1 timeout 1500 python bench.py --steps 1 --warmup 3 > gpurun_out/r2g_bench_sharded_w1.json 2> gpurun_out/r2g_bench_sharded_w1.err; echo "sharded world-1 rc=$?"
cut -c1-1400 gpurun_out/r2g_bench.json
