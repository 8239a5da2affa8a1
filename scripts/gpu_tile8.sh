export GOAT_SK_VERBOSE=1
timeout 900 python scripts/sk_scan.py gpurun_out/tile8.json "1000,fp32" "1000,fp32,GOAT_SK_TILE_CL=8" "2000,fp32,GOAT_SK_TILE_CL=8" "504,fp32,GOAT_SK_TILE_CL=8" > gpurun_out/tile8.log 2>&1; cut -c1-200 gpurun_out/tile8.log
