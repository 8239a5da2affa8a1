nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/g_smoke.log
timeout 1500 python -m pytest tests/ -q -m gpu --timeout 300 -p no:cacheprovider -rf > gpurun_out/g_pytest.log 2>&1; echo "pytest rc=$?"; grep -E "passed|failed|FAILED" gpurun_out/g_pytest.log | tail -5
timeout 900 python bench.py > gpurun_out/g_bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/g_bench.log | cut -c1-300
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/g_bench_ref.log 2>&1; echo "ref rc=$?"; tail -1 gpurun_out/g_bench_ref.log | cut -c1-200
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --steps 3 --warmup 3 > gpurun_out/g_bench_torchrun.log 2>&1; echo "torchrun bench rc=$?"; tail -1 gpurun_out/g_bench_torchrun.log | cut -c1-200
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29512 bench.py --impl reference --gpus 1 --steps 2 --warmup 1 > gpurun_out/g_ref_torchrun.log 2>&1; echo "torchrun ref rc=$?"; tail -1 gpurun_out/g_ref_torchrun.log | cut -c1-200
GOAT_BENCH_C5=0 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/g_launches.csv python bench.py --steps 2 --warmup 3 > gpurun_out/g_ncu.log 2>&1; echo "ncu rc=$?"
