# ncu of the persistent LOT kernel at n=1000 fp32, 16 CTAs (band-bound) and default CTAs
python scripts/prof_sweep.py 1000 fp32 50 > gpurun_out/prof_plain.log 2>&1 && \
GOAT_SK_BLOCKS=16 ncu --set full --import-source on --clock-control none -k regex:sk_persistent -c 1 -o gpurun_out/sk_n1000_b16 python scripts/prof_sweep.py 1000 fp32 50 > gpurun_out/ncu1.log 2>&1; echo "ncu1 rc=$?"
ncu --set full --import-source on --clock-control none -k regex:sk_persistent -c 1 -o gpurun_out/sk_n1000_b148 python scripts/prof_sweep.py 1000 fp32 50 > gpurun_out/ncu2.log 2>&1; echo "ncu2 rc=$?"
cat gpurun_out/prof_plain.log
