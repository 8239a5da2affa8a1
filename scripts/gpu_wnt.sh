timeout 1500 python scripts/sk_scan.py gpurun_out/sk_scan_wnt.json \
 "10000,fp32," "10000,fp32,GOAT_SK_WNT=256" "20000,fp32," "20000,fp32,GOAT_SK_WNT=256" "20000,fp32,GOAT_SK_WNT=256;GOAT_SK_MAXCH=4" \
 "40000,fp32," "40000,fp32,GOAT_SK_WNT=256" "40000,fp32,GOAT_SK_WNT=256;GOAT_SK_STAGES=4" "65536,fp32," "65536,fp32,GOAT_SK_WNT=256" \
 "10000,fp64," "10000,fp64,GOAT_SK_WNT=256" "20000,fp64," "20000,fp64,GOAT_SK_WNT=256"
timeout 600 env GOAT_SK_WNT=256 python -m pytest tests/test_lot_large_gpu.py -q -x -p no:cacheprovider 2>&1 | tail -2
