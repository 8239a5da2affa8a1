nvidia-smi --query-gpu=name,clocks.sm --format=csv,noheader
timeout 1200 python -m pytest tests/test_csr_gpu.py -q -x -m gpu -p no:cacheprovider > gpurun_out/csr_pytest.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/csr_pytest.log
timeout 900 python scripts/prof_spmm.py 10000 3 > gpurun_out/spmm.log 2>&1; echo "spmm10k rc=$?"
timeout 900 python scripts/prof_spmm.py 20000 3 >> gpurun_out/spmm.log 2>&1; echo "spmm20k rc=$?"
timeout 1200 python scripts/prof_spmm.py 40000 2 >> gpurun_out/spmm.log 2>&1; echo "spmm40k rc=$?"
cat gpurun_out/spmm.log | tail -5
