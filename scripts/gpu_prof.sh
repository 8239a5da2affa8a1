export GOAT_SK_BLOCKS=64
python scripts/prof_sweep.py 1000 fp32 50 > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:sk_persistent -c 1 -o gpurun_out/sk_n1000 python scripts/prof_sweep.py 1000 fp32 50 > gpurun_out/ncu.log 2>&1
echo "ncu rc=$?"; tail -3 gpurun_out/ncu.log; cat gpurun_out/prof_plain.log
