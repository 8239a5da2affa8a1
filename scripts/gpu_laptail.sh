# auction phase tail scan (GOAT_LAP_TAIL: a phase ends at n/div unassigned rows)
for div in ${DIVS:-512 128 64 32 16}; do
  echo "== TAIL=$div"
  GOAT_LAP_TAIL=$div GOAT_LAP_VERBOSE=1 timeout 300 python scripts/run_configs.py 4,4,3,3 2>&1 | python -c "
import sys, json
for l in sys.stdin:
    l = l.strip()
    if l.startswith('{'):
        d = json.loads(l); print('  cfg', d['config'], 'lap_ms', d['phase_ms']['lap'], 'total_ms', d['phase_ms']['total'], 'obj', d['objective'])
    elif 'n=2000' in l or 'n=5000' in l: print('  ', l)
"
done > gpurun_out/laptail${SUF:-}.log
echo rc=$?
