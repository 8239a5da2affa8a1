bash scripts/gpu_round.sh
timeout 900 python scripts/run_c5.py 30 40000 fp32 csr > gpurun_out/c5_csr_30.log 2>&1; echo "c5 rc=$?"; tail -3 gpurun_out/c5_csr_30.log
