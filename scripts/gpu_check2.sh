timeout 900 python -m pytest tests/ -q -m gpu -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log; grep FAILED gpurun_out/pytest_gpu.log | head
timeout 900 python scripts/sk_scan.py gpurun_out/sk_scan_final.json "1000,fp32," "1000,fp64," "2000,fp32," "5000,fp32," "10000,fp32," "20000,fp32," "40000,fp32," "5000,fp64," "20000,fp64,"
timeout 600 python bench.py > gpurun_out/bench.log 2>&1; tail -c 600 gpurun_out/bench.log
