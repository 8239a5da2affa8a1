export GOAT_SK_VERBOSE=1
timeout 900 python scripts/sk_scan.py gpurun_out/r2.json "4000,fp32" "4500,fp32" "5000,fp32" "6000,fp32" "6144,fp32,GOAT_SK_PIPE_R1=1" > gpurun_out/r2.log 2>&1; cut -c1-200 gpurun_out/r2.log
timeout 900 python -m pytest tests/test_lot_large_gpu.py tests/test_parity_gpu.py -q -m gpu --timeout 240 -p no:cacheprovider > gpurun_out/r2_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r2_pytest.log
timeout 600 python scripts/run_configs.py 3 2>&1 | cut -c1-300
