#!/bin/bash
# fp64-finish re-check, reference suite, c5 fp64-as-oracle, sharded bench at world 1, compute-sanitizer
cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests/test_parity_gpu.py tests/test_full_configs_gpu.py tests/test_wide_gpu.py -q -p no:cacheprovider > gpurun_out/r2i_tests.log 2>&1
tail -5 gpurun_out/r2i_tests.log
timeout 600 python scripts/fp32_status.py fp32 > gpurun_out/r2i_fp32.jsonl 2> gpurun_out/r2i_fp32.err
bash scripts/conformance.sh > gpurun_out/r2i_conformance.log 2>&1
tail -8 gpurun_out/r2i_conformance.log
timeout 1500 python scripts/c5_fp64_oracle.py > gpurun_out/r2i_c5_fp64_oracle.json 2> gpurun_out/r2i_c5_fp64_oracle.err; echo "c5 oracle rc=$?"
GOAT_BENCH_SHARDED=1 timeout 1500 python bench.py --steps 1 --warmup 3 > gpurun_out/r2i_bench_sharded_w1.json 2> gpurun_out/r2i_bench_sharded_w1.err; echo "sharded rc=$?"
for tool in racecheck synccheck memcheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python -m pytest tests/test_parity_gpu.py -q -p no:cacheprovider -x -k "c1_r0 or c4s_r0 or unif50 or faq_w300" > gpurun_out/r2i_sanitizer_$tool.log 2>&1
  echo "$tool rc=$?"; grep -c "ERROR SUMMARY\|Race reported\|Error:" gpurun_out/r2i_sanitizer_$tool.log; tail -3 gpurun_out/r2i_sanitizer_$tool.log
done
