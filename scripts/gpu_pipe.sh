nvidia-smi --query-gpu=name,clocks.sm --format=csv,noheader
GOAT_SK_PIPE_CL=3 timeout 900 python -m pytest tests/test_lot_large_gpu.py -q -x -m gpu -p no:cacheprovider > gpurun_out/pipe_pytest.log 2>&1; echo "pytest(cl=3) rc=$?"; tail -2 gpurun_out/pipe_pytest.log
export GOAT_SK_VERBOSE=1
timeout 1200 python scripts/sk_scan.py gpurun_out/pipe_scan.json \
  "20000,fp32" "20000,fp32,GOAT_SK_PIPE_CL=3" "24000,fp32" "24000,fp32,GOAT_SK_PIPE=0" "30000,fp32" "30000,fp32,GOAT_SK_PIPE=0" \
  "40000,fp32" "40000,fp32,GOAT_SK_PIPE_CL=4" "40000,fp32,GOAT_SK_PIPE_CL=6" "40000,fp32,GOAT_SK_PIPE=0" "65536,fp32,GOAT_SK_PIPE=2" "65536,fp32" > gpurun_out/pipe_scan.log 2>&1; echo "scan rc=$?"
cut -c1-230 gpurun_out/pipe_scan.log
