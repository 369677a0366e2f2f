#!/usr/bin/env bash
# A/B helper: ordered kernel round statistics at 2^24..2^28 + ordered parity tests
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_tcf_gpu.py tests/test_full_size_gpu.py -x -q -k "bit_exact or c1_full or 2p24 or c3" > gpurun_out/pytest_ab.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_ab.log
timeout 300 python scripts/ord_tune.py --log-slots 24 26 28 --cfg default > gpurun_out/ab.jsonl 2>/dev/null
python -c "
import json
for l in open('gpurun_out/ab.jsonl'):
    d=json.loads(l); print(d['log_slots'], *['%s %.2fG/s us/r=%.1f'%(op[:3],d[op]['g_ops_per_s'],d[op]['us_per_round']) for op in ('insert','delete')])"
