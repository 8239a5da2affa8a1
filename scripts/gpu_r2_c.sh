#!/bin/bash
# ncu of the 2-CTA wide-row Sinkhorn kernel at n = 40000 (4 sweeps)
cd $GRAFT_REPO_ROOT
mkdir -p /tmp/ncu
GOAT_SK_STAGES=6 python scripts/prof_sweep.py 40000 fp32 4 > gpurun_out/r2c_plain.log 2>&1
GOAT_SK_STAGES=6 ncu -f --set full --import-source on --clock-control none -k regex:sk_wide -c 1 -o /tmp/ncu/wide40k python scripts/prof_sweep.py 40000 fp32 4 > gpurun_out/r2c_ncu.log 2>&1; echo "ncu rc=$?"
python scripts/ncu_summary.py /tmp/ncu/wide40k.ncu-rep "sk_wide_kernel n=40000" > gpurun_out/r2c_summary.md 2>&1
python scripts/ncu_lines.py /tmp/ncu/wide40k.ncu-rep 40 > gpurun_out/r2c_lines.txt 2>&1
ncu -i /tmp/ncu/wide40k.ncu-rep --page details --csv > gpurun_out/r2c_details.csv 2>&1
ncu -i /tmp/ncu/wide40k.ncu-rep --page raw --csv > gpurun_out/r2c_raw.csv 2>&1
ncu -i /tmp/ncu/wide40k.ncu-rep --page source --csv --print-source sass > /tmp/ncu/sass.csv 2>&1; python scripts/sass_hot.py /tmp/ncu/sass.csv > gpurun_out/r2c_sass_hot.txt 2>&1

