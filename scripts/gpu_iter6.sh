#!/usr/bin/env bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_tcf_gpu.py -x -q -k "bit_exact or tunables or c1_full" > gpurun_out/pytest_tcf.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_tcf.log
show() { python -c "
import json
for l in open('$1'):
    d=json.loads(l); print('$2', d['log_slots'], d['cfg'], *['%s %.2fG/s r=%d us/r=%.1f carried=%d'%(op[:3],d[op]['g_ops_per_s'],d[op]['rounds'],d[op]['us_per_round'],d[op]['carried']) for op in ('insert','delete')])"; }
FK_ORD_ONEBAR=1 timeout 900 python scripts/ord_tune.py --log-slots 24 28 --cfg default "W=400000" "RS=1" "RS=1,W=400000" "RS=0,W=400000" "CTAS=3,W=400000" > gpurun_out/ob1.jsonl 2>/dev/null; show gpurun_out/ob1.jsonl ob1
