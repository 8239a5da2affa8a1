# final gate of the session: smoke, full GPU suite, bench, reference arm, launch list, c1/c4/c3 solves
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/z_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/z_smoke.log
timeout 1500 python -m pytest tests/ -q -m gpu --timeout 300 -p no:cacheprovider -rf > gpurun_out/z_pytest.log 2>&1; echo "pytest rc=$?"; grep -E "passed|failed|FAILED" gpurun_out/z_pytest.log | tail -5
timeout 900 python bench.py > gpurun_out/z_bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/z_bench.log | cut -c1-300
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/z_bench_ref.log 2>&1; echo "ref rc=$?"; tail -1 gpurun_out/z_bench_ref.log | cut -c1-200
GOAT_BENCH_C5=0 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/z_launches.csv python bench.py --steps 2 --warmup 3 > gpurun_out/z_ncu.log 2>&1; echo "ncu rc=$?"
timeout 600 python scripts/run_configs.py 1,4,3 > gpurun_out/z_configs.log 2>&1; echo "configs rc=$?"; cut -c1-250 gpurun_out/z_configs.log
