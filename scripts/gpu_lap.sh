timeout 1200 python -m pytest tests/test_lap_auction_gpu.py tests/test_parity_gpu.py -q -m gpu -p no:cacheprovider -k "lap or auction" > gpurun_out/pytest_lap.log 2>&1; tail -3 gpurun_out/pytest_lap.log; grep -E "FAILED|Error" gpurun_out/pytest_lap.log | head
timeout 1200 python scripts/run_configs.py 4,3
