export GOAT_SK_VERBOSE=1
timeout 900 python scripts/sk_scan.py gpurun_out/t256.json "64,fp32" "504,fp32" "1000,fp32" "2000,fp32" "1000,fp64" > gpurun_out/t256.log 2>&1; cut -c1-170 gpurun_out/t256.log
