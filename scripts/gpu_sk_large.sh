for n in 5000 10000 20000 40000; do python scripts/prof_sweep.py $n fp32 20; done
GOAT_SK_WIDE=1 python scripts/prof_sweep.py 5000 fp32 20
timeout 900 python -m pytest tests/ -q -m gpu -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log; grep FAILED gpurun_out/pytest_gpu.log | head
