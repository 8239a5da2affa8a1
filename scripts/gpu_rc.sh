set -x
timeout 900 python -m pytest tests/ -q -m gpu -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log; grep -E "FAILED|Error" gpurun_out/pytest_gpu.log | head
timeout 1500 python scripts/sk_scan.py gpurun_out/sk_scan_rc.json \
 "1000,fp32," "1000,fp32,GOAT_SK_RC=0" "1000,fp64," "1000,fp64,GOAT_SK_RC=0" "600,fp32," "600,fp32,GOAT_SK_RC=0" \
 "1500,fp32," "1500,fp32,GOAT_SK_RC=0" "2000,fp32," "2000,fp32,GOAT_SK_RC=0" "3000,fp32," "3000,fp32,GOAT_SK_RC=0" \
 "5000,fp32," "5000,fp32,GOAT_SK_RC=0" "8000,fp32," "8000,fp32,GOAT_SK_RC=0" "2000,fp64," "2000,fp64,GOAT_SK_RC=0" "4000,fp64," "4000,fp64,GOAT_SK_RC=0"
