export GOAT_SK_NOCOOP=1
python scripts/prof_sweep.py 10000 fp32 10 > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:sk_persistent -c 1 -o gpurun_out/sk_n10000 python scripts/prof_sweep.py 10000 fp32 10 > gpurun_out/ncu1.log 2>&1; echo "ncu1 rc=$?"
python scripts/prof_sweep.py 40000 fp32 3 >> gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:sk_persistent -c 1 -o gpurun_out/sk_n40000 python scripts/prof_sweep.py 40000 fp32 3 > gpurun_out/ncu2.log 2>&1; echo "ncu2 rc=$?"
cat gpurun_out/prof_plain.log
