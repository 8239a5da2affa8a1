export GOAT_SK_VERBOSE=1
timeout 900 python scripts/sk_scan.py gpurun_out/r1.json "3000,fp32" "3000,fp32,GOAT_SK_PIPE=3;GOAT_SK_PIPE_R1=2" "5000,fp32" "5000,fp32,GOAT_SK_PIPE=3;GOAT_SK_PIPE_R1=2" "8192,fp32" "8192,fp32,GOAT_SK_PIPE_R1=2" "10000,fp32,GOAT_SK_PIPE_R1=2" > gpurun_out/r1.log 2>&1; cut -c1-200 gpurun_out/r1.log
