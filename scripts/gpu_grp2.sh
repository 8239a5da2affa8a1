# tile kernel: row-group count scan at small n (GOAT_SK_TILE_GRP)
A=()
for n in 96 200; do for g in 0 4 6 8 12 16; do A+=("$n,fp64,GOAT_SK_TILE_GRP=$g"); A+=("$n,fp32,GOAT_SK_TILE_GRP=$g"); done; done
for n in 296 504 752; do for g in 0 8 12 16 24; do A+=("$n,fp64,GOAT_SK_TILE_GRP=$g"); A+=("$n,fp32,GOAT_SK_TILE_GRP=$g"); done; done
python scripts/sk_scan.py gpurun_out/grp_scan2.json "${A[@]}"
