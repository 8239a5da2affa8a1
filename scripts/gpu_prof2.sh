export GOAT_SK_NOCOOP=1
python scripts/prof_sweep.py 20000 fp32 5 > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:sk_persistent -c 1 -o gpurun_out/sk_tma_n20000 python scripts/prof_sweep.py 20000 fp32 5 > gpurun_out/ncu1.log 2>&1; echo "ncu1 rc=$?"
cat gpurun_out/prof_plain.log; tail -3 gpurun_out/ncu1.log
