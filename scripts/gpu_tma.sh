set -x
timeout 600 python -m pytest tests/test_lot_large_gpu.py -q -x -p no:cacheprovider > gpurun_out/pytest_large.log 2>&1; tail -3 gpurun_out/pytest_large.log
timeout 1200 python scripts/sk_scan.py gpurun_out/sk_scan_tma.json \
 "10000,fp32," "10000,fp32,GOAT_SK_TMA=0" "10000,fp32,GOAT_SK_STAGES=3" "10000,fp32,GOAT_SK_STAGES=4" \
 "20000,fp32," "20000,fp32,GOAT_SK_TMA=0" "20000,fp32,GOAT_SK_MAXCH=4" \
 "40000,fp32," "40000,fp32,GOAT_SK_TMA=0" "40000,fp32,GOAT_SK_MAXCH=4" "40000,fp32,GOAT_SK_MAXCH=3" "40000,fp32,GOAT_SK_STAGES=4" \
 "10000,fp64," "10000,fp64,GOAT_SK_TMA=0" "20000,fp64," "65536,fp32,"
timeout 900 python -m pytest tests/ -q -m gpu -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
