# ncu evidence for the round-1 kernels (summaries written on the box; reports stay in /tmp)
mkdir -p /tmp/ncu
export GOAT_SK_NOCOOP=1
python scripts/prof_sweep.py 40000 fp32 3 > gpurun_out/p3_plain.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:sk_pipe -c 1 -o /tmp/ncu/pipe40k python scripts/prof_sweep.py 40000 fp32 3 > gpurun_out/p3_ncu1.log 2>&1; echo "ncu pipe rc=$?"
python scripts/ncu_summary.py /tmp/ncu/pipe40k.ncu-rep "sk_pipe_kernel n=40000 fp32 (cluster 4, 3 sweeps + pre-check + row pass)" > gpurun_out/p3_pipe40k.md 2>&1
ncu -i /tmp/ncu/pipe40k.ncu-rep --page source --csv --print-source sass > /tmp/ncu/pipe40k_sass.csv 2>&1; python scripts/sass_hot.py /tmp/ncu/pipe40k_sass.csv 20 > gpurun_out/p3_pipe40k_sass.txt 2>&1
python scripts/prof_sweep.py 12288 fp32 20 >> gpurun_out/p3_plain.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:sk_pipe -c 1 -o /tmp/ncu/pipe12k python scripts/prof_sweep.py 12288 fp32 20 > gpurun_out/p3_ncu2.log 2>&1; echo "ncu pipe12k rc=$?"
python scripts/ncu_summary.py /tmp/ncu/pipe12k.ncu-rep "sk_pipe_kernel n=12288 fp32 (whole rows, 20 sweeps)" > gpurun_out/p3_pipe12k.md 2>&1
unset GOAT_SK_NOCOOP
python scripts/prof_spmm_one.py 20000 >> gpurun_out/p3_plain.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:spmm_t -c 2 -o /tmp/ncu/spmm20k python scripts/prof_spmm_one.py 20000 > gpurun_out/p3_ncu3.log 2>&1; echo "ncu spmm rc=$?"
python scripts/ncu_summary.py /tmp/ncu/spmm20k.ncu-rep "spmm_t_kernel n=20000 (config-5 law CSR, symmetric: A.Q then B.X^T)" > gpurun_out/p3_spmm20k.md 2>&1
GOAT_BENCH_C5=0 python bench.py --steps 2 --warmup 3 > gpurun_out/p3_bench.log 2>&1; echo "bench rc=$?"
GOAT_BENCH_C5=0 ncu --metrics gpu__time_duration.sum --clock-control none -c 500 --csv --log-file gpurun_out/p3_launches.csv python bench.py --steps 2 --warmup 3 > gpurun_out/p3_ncu4.log 2>&1; echo "ncu launches rc=$?"
cat gpurun_out/p3_plain.log
