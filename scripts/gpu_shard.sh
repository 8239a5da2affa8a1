timeout 1200 python -m pytest tests/test_sharded_gpu.py -q -x -p no:cacheprovider > gpurun_out/pytest_shard.log 2>&1; tail -25 gpurun_out/pytest_shard.log
