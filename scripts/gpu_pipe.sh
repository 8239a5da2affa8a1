nvidia-smi --query-gpu=name,clocks.sm --format=csv,noheader
GOAT_SK_PIPE_R=2 GOAT_SK_PIPE=2 timeout 900 python -m pytest tests/test_lot_large_gpu.py -q -x -m gpu -p no:cacheprovider > gpurun_out/pipe_pytest.log 2>&1; echo "pytest(R=2) rc=$?"; tail -2 gpurun_out/pipe_pytest.log
timeout 900 python -m pytest tests/test_lot_large_gpu.py -q -x -m gpu -p no:cacheprovider > gpurun_out/pipe_pytest1.log 2>&1; echo "pytest(default) rc=$?"; tail -2 gpurun_out/pipe_pytest1.log
export GOAT_SK_VERBOSE=1
timeout 1200 python scripts/sk_scan.py gpurun_out/pipe_scan.json \
  "12288,fp32" "20000,fp32" "20000,fp32,GOAT_SK_PIPE_R=2" "20000,fp32,GOAT_SK_PIPE_R=2;GOAT_SK_PIPE_CL=4" \
  "40000,fp32" "40000,fp32,GOAT_SK_PIPE_R=2" "40000,fp32,GOAT_SK_PIPE_R=2;GOAT_SK_PIPE_CL=8" "40000,fp32,GOAT_SK_PIPE_R=2;GOAT_SK_RES=2" \
  "65536,fp32" "65536,fp32,GOAT_SK_PIPE_R=2;GOAT_SK_PIPE=2" > gpurun_out/pipe_scan.log 2>&1; echo "scan rc=$?"
cut -c1-230 gpurun_out/pipe_scan.log
