set -o pipefail
python scripts/prof_gemm.py 5000 sym > gpurun_out/prof_gemm_plain.log 2>&1 && cat gpurun_out/prof_gemm_plain.log && \
ncu --set full --import-source on --clock-control none -k regex:tc_gemm -c 2 -o gpurun_out/tc_gemm_n5000 python scripts/prof_gemm.py 5000 sym > gpurun_out/ncu_gemm.log 2>&1; echo "ncu gemm rc=$?"
python scripts/prof_sweep.py 5000 fp32 20 > gpurun_out/prof_sk5000_plain.log 2>&1 && cat gpurun_out/prof_sk5000_plain.log && \
ncu --set full --import-source on --clock-control none -k regex:sk_persistent -c 1 -o gpurun_out/sk_n5000 python scripts/prof_sweep.py 5000 fp32 20 > gpurun_out/ncu_sk5000.log 2>&1; echo "ncu sk5000 rc=$?"
python scripts/prof_sweep.py 1000 fp32 50 > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:sk_persistent -c 1 -o gpurun_out/sk_n1000 python scripts/prof_sweep.py 1000 fp32 50 > gpurun_out/ncu_sk1000.log 2>&1; echo "ncu sk1000 rc=$?"
python bench.py --steps 2 --warmup 3 > gpurun_out/bench_plain.log 2>&1 && tail -1 gpurun_out/bench_plain.log && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 > gpurun_out/ncu_bench.log 2>&1; echo "ncu launches rc=$?"
