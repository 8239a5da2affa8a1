timeout 900 python -m pytest tests/test_lap_auction_gpu.py -q -x -m gpu -p no:cacheprovider > gpurun_out/lap_pytest.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/lap_pytest.log
GOAT_LAP_VERBOSE=1 timeout 900 python scripts/run_c5.py 5 40000 fp32 csr > gpurun_out/c5_lap.log 2>&1; echo "c5 rc=$?"; tail -4 gpurun_out/c5_lap.log
