set -x
timeout 900 python -m pytest tests/ -q -m gpu -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 1200 python scripts/sk_scan.py gpurun_out/sk_scan.json \
 "1000,fp32," "1000,fp32,GOAT_SK_RES=0" "1000,fp64," "1000,fp64,GOAT_SK_RES=0" "600,fp32," "600,fp32,GOAT_SK_RES=0" "2000,fp32," \
 "10000,fp32," "10000,fp32,GOAT_SK_MAXCH=4" "10000,fp32,GOAT_SK_MAXCH=3" \
 "20000,fp32," "20000,fp32,GOAT_SK_MAXCH=4" "20000,fp32,GOAT_SK_MAXCH=3" \
 "40000,fp32," "40000,fp32,GOAT_SK_MAXCH=4" "40000,fp32,GOAT_SK_MAXCH=3" \
 "5000,fp64," "10000,fp64," "10000,fp64,GOAT_SK_MAXCH=4" "10000,fp64,GOAT_SK_MAXCH=3"
