#!/usr/bin/env bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
show() { python -c "
import json
for l in open('$1'):
    d=json.loads(l); print(d['log_slots'], d['cfg'], 'rs', d['rs'], *['%s %.2fG/s r=%d us/r=%.1f'%(op[:3],d[op]['g_ops_per_s'],d[op]['rounds'],d[op]['us_per_round']) for op in ('insert','delete')])"; }
timeout 600 python scripts/ord_tune.py --log-slots 24 26 --cfg default "CTAS=4" "CTAS=4,W=262144" "CTAS=3,W=262144" "W=262144" "RS=1,W=262144" "CTAS=4,RS=1,W=262144" > gpurun_out/t24.jsonl 2>/dev/null; show gpurun_out/t24.jsonl
