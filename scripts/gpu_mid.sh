export GOAT_SK_VERBOSE=1
timeout 900 python scripts/sk_scan.py gpurun_out/mid_scan.json "6400,fp32" "6400,fp32,GOAT_SK_PIPE=0" "7168,fp32" "7168,fp32,GOAT_SK_PIPE=0" "8192,fp32" "10000,fp32" "12288,fp32" > gpurun_out/mid_scan.log 2>&1; echo "scan rc=$?"
cut -c1-200 gpurun_out/mid_scan.log
timeout 900 python -m pytest tests/test_lot_large_gpu.py tests/test_sharded_gpu.py -q -m gpu --timeout 240 -p no:cacheprovider > gpurun_out/mid_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/mid_pytest.log
