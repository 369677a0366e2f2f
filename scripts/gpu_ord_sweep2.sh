#!/usr/bin/env bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
for rs in 1 2 3; do for w in 65536 131072 262144 524288; do
  FK_ORD_RES_SHIFT=$rs FK_ORD_WINDOW=$w timeout 300 python bench.py --steps 2 --no-cpu --no-e2e --no-concurrent --no-launch-count > gpurun_out/sw.json 2>/dev/null
  python -c "
import json
d=json.load(open('gpurun_out/sw.json')); p=d['per_op']
print('rs=$rs W=$w', 'ins %.2f G/s'%(p['insert']['ops_per_s']/1e9), 'del %.2f G/s'%(p['delete']['ops_per_s']/1e9), 'qpos %.2f qneg %.2f'%(p['query_pos']['ops_per_s']/1e9, p['query_neg']['ops_per_s']/1e9), 'value %.3g'%d['value'])"
done; done
FK_ORD_RES_SHIFT=2 FK_ORD_WINDOW=262144 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_tcf -c 4 -o gpurun_out/prof_tcf_ordered2 -f python scripts/prof_tcf.py 28 ordered > gpurun_out/prof2.log 2>&1; echo "ncu rc=$?"
