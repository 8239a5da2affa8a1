nvidia-smi --query-gpu=name,clocks.sm --format=csv,noheader
timeout 1500 python -m pytest tests/ -q -m gpu --timeout 240 -p no:cacheprovider -rf > gpurun_out/tile_pytest.log 2>&1; echo "pytest rc=$?"; grep -E "passed|failed|FAILED|Error" gpurun_out/tile_pytest.log | tail -12
timeout 600 python bench.py --steps 5 > gpurun_out/tile_bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/tile_bench.log | cut -c1-900
