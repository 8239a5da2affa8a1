# re-entry verification: smoke, full GPU suite, bench, reference arm
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/v_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/v_smoke.log
timeout 1500 python -m pytest tests/ -q -m gpu --timeout 300 -p no:cacheprovider -rf > gpurun_out/v_pytest.log 2>&1; echo "pytest rc=$?"; grep -E "passed|failed|FAILED" gpurun_out/v_pytest.log | tail -5
timeout 900 python bench.py > gpurun_out/v_bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/v_bench.log | cut -c1-400
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/v_bench_ref.log 2>&1; echo "ref rc=$?"; tail -1 gpurun_out/v_bench_ref.log | cut -c1-300
