# 3-row bands for whole rows (GOAT_SK_PIPE_R1=3): parity at n=4501/5000 and per-sweep time
GOAT_SK_PIPE_R1=3 timeout 600 python -m pytest tests/test_lot_large_gpu.py -q -m gpu -p no:cacheprovider -k "4501 or 5000" > gpurun_out/r3_pytest.log 2>&1; echo "pytest r3 rc=$?"; tail -2 gpurun_out/r3_pytest.log
A=()
for n in 4200 4501 5000 5400 6000; do A+=("$n,fp32,GOAT_SK_PIPE_R1=2"); A+=("$n,fp32,GOAT_SK_PIPE_R1=3"); done
A+=("5000,fp32,GOAT_SK_PIPE_R1=2" "5000,fp32,GOAT_SK_PIPE_R1=3")
python scripts/sk_scan.py gpurun_out/r3_scan.json "${A[@]}"
