export GOAT_SK_NOCOOP=1
mkdir -p /tmp/ncu
ncu --set full --import-source on --clock-control none -k regex:sk_pipe -c 1 -o /tmp/ncu/pipe_n20000 python scripts/prof_sweep.py 20000 fp32 4 > gpurun_out/pipe_ncu1.log 2>&1; echo "ncu1 rc=$?"
python scripts/ncu_summary.py /tmp/ncu/pipe_n20000.ncu-rep "pipe n=20000 S=5" > gpurun_out/pipe_n20000_summary.md 2>&1
python scripts/ncu_lines.py /tmp/ncu/pipe_n20000.ncu-rep 40 > gpurun_out/pipe_n20000_lines.txt 2>&1
ncu -i /tmp/ncu/pipe_n20000.ncu-rep --page details --csv > gpurun_out/pipe_n20000_details.csv 2>&1
ncu -i /tmp/ncu/pipe_n20000.ncu-rep --page source --csv --print-source sass > gpurun_out/pipe_n20000_sass.csv 2>&1
ls -la gpurun_out
