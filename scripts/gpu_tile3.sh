export GOAT_SK_VERBOSE=1
timeout 900 python scripts/sk_scan.py gpurun_out/tile_scan4.json "1000,fp32" "1000,fp32,GOAT_SK_TILE_MERGE=8" "1000,fp32,GOAT_SK_TILE_GROUPS=16" "1000,fp32,GOAT_SK_TILE_GROUPS=24" "2000,fp32" "2000,fp32,GOAT_SK_TILE_MERGE=8" "2000,fp32,GOAT_SK_TILE_GROUPS=24" > gpurun_out/tile_scan4.log 2>&1; echo "scan rc=$?"
cut -c1-200 gpurun_out/tile_scan4.log
