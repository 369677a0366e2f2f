#!/usr/bin/env bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
show() { python -c "
import json
for l in open('$1'):
    d=json.loads(l); print('$2', d['log_slots'], *['%s %.2fG/s us/r=%.1f'%(op[:3],d[op]['g_ops_per_s'],d[op]['us_per_round']) for op in ('insert','delete')])"; }
for sp in 0 2; do FK_ORD_SPEC=$sp timeout 300 python scripts/ord_tune.py --log-slots 24 26 28 --cfg default > gpurun_out/sp$sp.jsonl 2>/dev/null; show gpurun_out/sp$sp.jsonl spec$sp; done
FK_ORD_SPEC=2 timeout 300 python -m pytest tests/test_tcf_gpu.py -x -q -k "bit_exact" 2>&1 | tail -1
timeout 300 python -m pytest tests/test_gqf_gpu.py -x -q -k "capacity" 2>&1 | tail -1
