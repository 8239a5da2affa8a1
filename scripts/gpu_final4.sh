# gate after the auction tail default change: smoke, GPU suite, configs (steady state), bench
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/q_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/q_smoke.log
timeout 1500 python -m pytest tests/ -q -m gpu --timeout 300 -p no:cacheprovider -rf > gpurun_out/q_pytest.log 2>&1; echo "pytest rc=$?"; grep -E "passed|failed|FAILED" gpurun_out/q_pytest.log | tail -5
timeout 600 python scripts/run_configs.py 1,1,4,4,3,3 > gpurun_out/q_configs.log 2>&1; echo "configs rc=$?"
timeout 900 python bench.py > gpurun_out/q_bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/q_bench.log | cut -c1-250
