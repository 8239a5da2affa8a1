#!/bin/bash
# ncu: the fp64 Sinkhorn sweep at n = 40000 (fp64 finish of fp32 handles) and the tcgen05 gradient launch lists
cd $GRAFT_REPO_ROOT
mkdir -p /tmp/ncu
python scripts/prof_sweep.py 40000 fp64 3 > gpurun_out/r2p_plain64.log 2>&1; cat gpurun_out/r2p_plain64.log
python scripts/prof_sweep.py 5000 fp64 50 >> gpurun_out/r2p_plain64.log 2>&1
timeout 900 ncu -f --set full --import-source on --clock-control none -k regex:sk_persistent -c 1 -o /tmp/ncu/p64 python scripts/prof_sweep.py 40000 fp64 2 > gpurun_out/r2p_ncu64.log 2>&1; echo "ncu rc=$?"
python scripts/ncu_summary.py /tmp/ncu/p64.ncu-rep "sk_persistent_kernel<double> n=40000" > gpurun_out/r2p_ncu_p64.md 2>&1
python scripts/ncu_lines.py /tmp/ncu/p64.ncu-rep 30 > gpurun_out/r2p_ncu_p64_lines.txt 2>&1
ncu -i /tmp/ncu/p64.ncu-rep --page details --csv > gpurun_out/r2p_ncu_p64_details.csv 2>&1
for a in "5000 sym" "2000 dir" "8192 sym"; do
  python scripts/prof_gemm.py $a
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2p_gemm_$(echo $a | tr ' ' '_').csv python scripts/prof_gemm.py $a > /dev/null 2>&1
done
