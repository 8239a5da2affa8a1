export GOAT_SK_VERBOSE=1
timeout 900 python scripts/sk_scan.py gpurun_out/tile_scan3.json "64,fp32" "504,fp32" "1000,fp32" "2000,fp32" "1000,fp64" "2000,fp64" > gpurun_out/tile_scan3.log 2>&1; echo "scan rc=$?"
cut -c1-220 gpurun_out/tile_scan3.log
