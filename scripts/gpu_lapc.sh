# warm-started LAP repair: one CTA (default below 200 KB of state) vs the 16-CTA cluster, c4/c3 steady state
GOAT_LAP_VERBOSE=1 timeout 300 python scripts/run_configs.py 4,4,3,3 > gpurun_out/lapc_default.log 2>&1; echo "default rc=$?"
GOAT_LAP_CLUSTER=2 GOAT_LAP_VERBOSE=1 timeout 300 python scripts/run_configs.py 4,4,3,3 > gpurun_out/lapc_cluster.log 2>&1; echo "cluster rc=$?"
