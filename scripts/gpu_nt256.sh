export GOAT_SK_VERBOSE=1
timeout 900 python scripts/sk_scan.py gpurun_out/nt256_scan.json "40000,fp32" "40000,fp32,GOAT_SK_PIPE_NT=256" "40000,fp32,GOAT_SK_PIPE_NT=256;GOAT_SK_PIPE_CL=4" "20000,fp32" "20000,fp32,GOAT_SK_PIPE_NT=256" "65536,fp32" "65536,fp32,GOAT_SK_PIPE_NT=256" > gpurun_out/nt256_scan.log 2>&1; echo "scan rc=$?"
cut -c1-220 gpurun_out/nt256_scan.log
GOAT_SK_PIPE_NT=256 timeout 900 python -m pytest tests/test_lot_large_gpu.py -q -x -m gpu --timeout 240 -p no:cacheprovider > gpurun_out/nt256_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/nt256_pytest.log
