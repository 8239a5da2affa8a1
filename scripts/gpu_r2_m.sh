#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 1500 python bench.py --steps 3 --warmup 3 > gpurun_out/r2m_bench.json 2> gpurun_out/r2m_bench.err; echo "bench rc=$?"
python - <<'PY'
import json
d=json.load(open('gpurun_out/r2m_bench.json'))
print(d['value'], d['e2e']['value'], d['roofline']['frac'])
for k,v in d['kernels'].items():
    if k.startswith('sinkhorn'): print(k, round(v['us'],1), round(v['frac_hbm'],3))
PY
