# bulk-copy ring with an L2 evict_last hint (GOAT_SK_L2HINT) vs without
A=()
for n in 4200 5000 5400 6000; do A+=("$n,fp32,GOAT_SK_L2HINT=0"); A+=("$n,fp32,GOAT_SK_L2HINT=1;GOAT_SK_L2HINT_MB=200"); done
A+=("8192,fp32,GOAT_SK_L2HINT=0" "8192,fp32,GOAT_SK_L2HINT=1;GOAT_SK_L2HINT_MB=400" "5000,fp32,GOAT_SK_L2HINT=0" "5000,fp32,GOAT_SK_L2HINT=1")
python scripts/sk_scan.py gpurun_out/l2hint_scan.json "${A[@]}"
