for c in 4 3; do
for lc in 1 2; do
echo "== config $c GOAT_LAP_CLUSTER=$lc"; GOAT_LAP_CLUSTER=$lc GOAT_LAP_VERBOSE=1 timeout 600 python scripts/run_configs.py $c 2>&1 | grep -E "repair|\"lap\"" | sed -E 's/.*"lap": ([0-9.]+).*/lap_ms=\1/' | tail -2
done; done
