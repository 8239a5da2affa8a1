export GOAT_SK_NOCOOP=1
python scripts/prof_sweep.py 40000 fp32 5 > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:sk_persistent -c 1 -o gpurun_out/sk_n40000 python scripts/prof_sweep.py 40000 fp32 5 > gpurun_out/ncu_sk40000.log 2>&1; echo "ncu rc=$?"; cat gpurun_out/prof_plain.log; tail -2 gpurun_out/ncu_sk40000.log
unset GOAT_SK_NOCOOP
timeout 900 python -m pytest tests/test_lot_large_gpu.py -q -m gpu -p no:cacheprovider 2>&1 | tail -2
