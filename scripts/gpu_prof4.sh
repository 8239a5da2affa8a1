mkdir -p /tmp/ncu
export GOAT_SK_NOCOOP=1
ncu --set full --import-source on --clock-control none -k regex:sk_pipe -c 1 -o /tmp/ncu/pipe12k python scripts/prof_sweep.py 12288 fp32 20 > gpurun_out/p4_ncu1.log 2>&1; echo "ncu pipe12k rc=$?"
python scripts/ncu_summary.py /tmp/ncu/pipe12k.ncu-rep "sk_pipe_kernel n=12288 fp32 (whole rows, fixed-shift sweeps, 20 sweeps)" > gpurun_out/p4_pipe12k.md 2>&1
GOAT_LAP_CLUSTER=2 ncu --set full --clock-control none -k regex:"lap_auction_kernel|lap_cluster_sap" -c 2 -o /tmp/ncu/lap5k python scripts/prof_lap.py 5000 > gpurun_out/p4_ncu2.log 2>&1; echo "ncu lap rc=$?"
python scripts/ncu_summary.py /tmp/ncu/lap5k.ncu-rep "device LAP n=5000 hub cost: auction (cooperative) + cluster repair" > gpurun_out/p4_lap5k.md 2>&1
head -40 gpurun_out/p4_lap5k.md
