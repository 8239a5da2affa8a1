#!/bin/bash
# round 2 gate: GPU suite, fp32 status, c5 bench (plain), ncu launch list of the same command, ncu --set full of the wide kernel
cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2g_smi.txt 2>&1
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider --durations=15 > gpurun_out/r2g_tests.log 2>&1
tail -3 gpurun_out/r2g_tests.log
timeout 600 python scripts/fp32_status.py fp32 > gpurun_out/r2g_fp32.jsonl 2> gpurun_out/r2g_fp32.err
timeout 1500 python bench.py --steps 2 --warmup 3 > gpurun_out/r2g_bench.json 2> gpurun_out/r2g_bench.err; echo "bench rc=$?"
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r2g_bench_ref.json 2> gpurun_out/r2g_bench_ref.err; echo "ref rc=$?"
GOAT_BENCH_SECONDARY=0 timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2g_launches.csv python bench.py --steps 1 --warmup 3 > gpurun_out/r2g_ncu_bench.log 2>&1; echo "ncu list rc=$?"
mkdir -p /tmp/ncu
python scripts/prof_sweep.py 40000 fp32 4 > gpurun_out/r2g_plain.log 2>&1
timeout 900 ncu -f --set full --import-source on --clock-control none -k regex:sk_wide -c 1 -o /tmp/ncu/wide40k python scripts/prof_sweep.py 40000 fp32 4 > gpurun_out/r2g_ncu.log 2>&1; echo "ncu full rc=$?"
python scripts/ncu_summary.py /tmp/ncu/wide40k.ncu-rep "sk_wide kernel n=40000" > gpurun_out/r2g_ncu_wide40k.md 2>&1
python scripts/ncu_lines.py /tmp/ncu/wide40k.ncu-rep 40 > gpurun_out/r2g_ncu_wide40k_lines.txt 2>&1
ncu -i /tmp/ncu/wide40k.ncu-rep --page raw --csv > gpurun_out/r2g_ncu_wide40k_raw.csv 2>&1
cut -c1-1500 gpurun_out/r2g_bench.json
