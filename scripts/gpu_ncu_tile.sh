export GOAT_SK_NOCOOP=1
mkdir -p /tmp/ncu
GOAT_BENCH_C5=0 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/f_launches.csv python bench.py --steps 2 --warmup 3 > gpurun_out/f_ncu.log 2>&1; echo "ncu launches rc=$?"
ncu --set full --import-source on --clock-control none -k regex:sk_tile -c 1 -o /tmp/ncu/tile1k python scripts/prof_sweep.py 1000 fp32 50 > gpurun_out/f_ncu2.log 2>&1; echo "ncu tile rc=$?"
python scripts/ncu_summary.py /tmp/ncu/tile1k.ncu-rep "sk_tile_kernel n=1000 fp32 (50 sweeps, one cooperative launch)" > gpurun_out/f_tile1k.md 2>&1
ncu -i /tmp/ncu/tile1k.ncu-rep --page source --csv --print-source sass > /tmp/ncu/t_sass.csv 2>&1; python scripts/sass_hot.py /tmp/ncu/t_sass.csv 20 > gpurun_out/f_tile1k_sass.txt 2>&1
tail -3 gpurun_out/f_ncu.log
