timeout 900 python scripts/gemm_err.py 2>&1 | tail -20
timeout 900 python -m pytest tests/test_gemm_gpu.py tests/test_parity_gpu.py -q -m gpu --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed|^FAILED" gpurun_out/pytest_gpu.log | tail -25
