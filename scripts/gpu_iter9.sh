#!/usr/bin/env bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_tcf_bulk_gpu.py tests/test_acceptance_gpu.py -q -x -k "bulk or c02 or c06 or c07" > gpurun_out/pytest_bulk.log 2>&1; echo "pytest chunked rc=$?"; tail -3 gpurun_out/pytest_bulk.log
FK_ROUTE=0 timeout 300 python -m pytest tests/test_tcf_bulk_gpu.py -q -x > gpurun_out/pytest_bulk0.log 2>&1; echo "pytest seq rc=$?"; tail -2 gpurun_out/pytest_bulk0.log
for r in 0 1; do FK_ROUTE=$r timeout 180 python bench.py --workload bulk_tcf --steps 5 --no-cpu --no-e2e > gpurun_out/bb$r.json 2>/dev/null; python -c "
import json
d=json.load(open('gpurun_out/bb$r.json')); print('route=$r value %.3g'%d['value'], {k:(round(v['ops_per_s']/1e9,3), round(v['ms'],2)) for k,v in d['per_op'].items()})"; done
