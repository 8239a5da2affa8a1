timeout 600 python -m pytest tests/test_lap_auction_gpu.py -q -x -m gpu -p no:cacheprovider > gpurun_out/lap3_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/lap3_pytest.log
for k in 0 1; do
GOAT_LAP_KEEP=$k GOAT_LAP_VERBOSE=1 timeout 600 python scripts/run_configs.py 3 2>&1 | grep -E "lap n=5000|config" | cut -c1-330
GOAT_LAP_KEEP=$k GOAT_LAP_VERBOSE=1 timeout 900 python scripts/run_c5.py 1 40000 fp32 csr 2>&1 | grep -E "lap n=40000|phase" | cut -c1-300
done
