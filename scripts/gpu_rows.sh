timeout 900 python scripts/sk_scan.py gpurun_out/sk_scan_rows.json \
 "1000,fp32,GOAT_SK_RC=0" "1000,fp32,GOAT_SK_RC=0;GOAT_SK_ROWS=4" "1000,fp32,GOAT_SK_RC=0;GOAT_SK_ROWS=2" \
 "600,fp32,GOAT_SK_RC=0" "600,fp32,GOAT_SK_RC=0;GOAT_SK_ROWS=4" "600,fp32,GOAT_SK_RC=0;GOAT_SK_ROWS=2" "1000,fp32," "1000,fp64,GOAT_SK_RC=0"
for r in 4 2; do GOAT_SK_RC=0 GOAT_SK_ROWS=$r GOAT_SK_TRACE=10 python scripts/prof_sweep.py 1000 fp32 50 2>&1 | grep -v Warn; done
