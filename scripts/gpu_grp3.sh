# after the small-n row-group cap: GPU suite, c1/c4 solves, smoke
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/w_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/w_smoke.log
timeout 1500 python -m pytest tests/ -q -m gpu --timeout 300 -p no:cacheprovider -rf -x > gpurun_out/w_pytest.log 2>&1; echo "pytest rc=$?"; grep -E "passed|failed|FAILED|Error" gpurun_out/w_pytest.log | tail -8
timeout 600 python scripts/run_configs.py 1,4 > gpurun_out/w_configs.log 2>&1; echo "configs rc=$?"; cut -c1-300 gpurun_out/w_configs.log
GOAT_SK_TILE_GRP=999 timeout 600 python scripts/run_configs.py 1 > gpurun_out/w_configs_old.log 2>&1; echo "configs(old grouping) rc=$?"; cut -c1-300 gpurun_out/w_configs_old.log
