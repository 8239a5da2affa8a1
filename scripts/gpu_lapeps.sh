# auction schedule scan: final eps exponent and theta (exact repair keeps the optimum)
for cfg in "7 8" "5 8" "4 8" "3 8" "7 16" "5 16" "4 16"; do
  set -- $cfg
  echo "== EPS_END=$1 THETA=$2"
  GOAT_LAP_EPS_END=$1 GOAT_LAP_THETA=$2 GOAT_LAP_VERBOSE=1 timeout 300 python scripts/run_configs.py 4,4,3,3 2>&1 | grep -E "n=(2000|5000)|^\{" | cut -c1-200
done > gpurun_out/lapeps.log
echo rc=$?
