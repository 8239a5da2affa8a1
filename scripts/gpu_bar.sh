export GOAT_SK_VERBOSE=1
timeout 900 python scripts/sk_scan.py gpurun_out/bar.json "64,fp32" "1000,fp32" "2000,fp32" "5000,fp32" "1000,fp64" > gpurun_out/bar.log 2>&1; cut -c1-160 gpurun_out/bar.log
timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_lot_large_gpu.py -q -m gpu --timeout 240 -p no:cacheprovider > gpurun_out/bar_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/bar_pytest.log
timeout 600 python bench.py --steps 5 > gpurun_out/bar_bench.log 2>&1; GOAT_BENCH_C5=0 echo; tail -1 gpurun_out/bar_bench.log | cut -c1-200
