# ncu --set full of the n=5000 fp32 LOT (2-row-band bulk-copy pipeline): is G L2-resident across sweeps?
export GOAT_SK_NOCOOP=1
mkdir -p /tmp/ncu
timeout 300 python scripts/prof_sweep.py 5000 fp32 20; echo "plain rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:sk_ -c 1 -o /tmp/ncu/sk5k python scripts/prof_sweep.py 5000 fp32 20 > gpurun_out/ncu5k.log 2>&1; echo "ncu rc=$?"
python scripts/ncu_summary.py /tmp/ncu/sk5k.ncu-rep "sk n=5000 fp32, 20 sweeps" > gpurun_out/sk5k_summary.md 2>&1
ncu -i /tmp/ncu/sk5k.ncu-rep --page raw --csv > gpurun_out/sk5k_raw.csv 2>&1
tail -3 gpurun_out/ncu5k.log
