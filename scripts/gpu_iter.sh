#!/usr/bin/env bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_tcf_gpu.py -x -q 2>&1 | tail -3
for rs in 1 2 3; do for w in 262144 524288; do
  FK_ORD_RES_SHIFT=$rs FK_ORD_WINDOW=$w timeout 300 python bench.py --steps 2 --no-cpu --no-e2e --no-concurrent --no-launch-count > gpurun_out/sw.json 2>/dev/null
  python -c "
import json
d=json.load(open('gpurun_out/sw.json')); p=d['per_op']
print('rs=$rs W=$w', 'ins %.2f G/s'%(p['insert']['ops_per_s']/1e9), 'del %.2f G/s'%(p['delete']['ops_per_s']/1e9), 'value %.3g'%d['value'])"
done; done
