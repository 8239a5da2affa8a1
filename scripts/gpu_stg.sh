export GOAT_SK_VERBOSE=1
timeout 900 python scripts/sk_scan.py gpurun_out/stg.json "504,fp32" "1000,fp32" "1000,fp32,GOAT_SK_TILE_STAGGER=0" "2000,fp32" "1000,fp64" > gpurun_out/stg.log 2>&1; cut -c1-170 gpurun_out/stg.log
