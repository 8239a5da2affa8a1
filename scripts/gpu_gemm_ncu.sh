mkdir -p /tmp/ncu
python scripts/prof_gemm.py 8192 sym > gpurun_out/g_plain.log 2>&1
python scripts/prof_gemm.py 5000 sym >> gpurun_out/g_plain.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:tc_gemm -c 1 -o /tmp/ncu/gemm8k python scripts/prof_gemm.py 8192 sym > gpurun_out/g_ncu.log 2>&1; echo "ncu rc=$?"
ncu -i /tmp/ncu/gemm8k.ncu-rep --page details --csv > gpurun_out/g_details.csv 2>&1
ncu -i /tmp/ncu/gemm8k.ncu-rep --page raw --csv > gpurun_out/g_raw.csv 2>&1
ncu -i /tmp/ncu/gemm8k.ncu-rep --page source --csv --print-source sass > /tmp/ncu/g_sass.csv 2>&1; python scripts/sass_hot.py /tmp/ncu/g_sass.csv 25 > gpurun_out/g_sass.txt 2>&1
cat gpurun_out/g_plain.log
timeout 600 python scripts/sk_scan.py gpurun_out/pipe_scan2.json "20000,fp32" "24000,fp32" "40000,fp32" "65536,fp32" > gpurun_out/pipe_scan2.log 2>&1; cut -c1-200 gpurun_out/pipe_scan2.log
