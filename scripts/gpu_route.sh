#!/usr/bin/env bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
FK_ROUTE_PREFIX=1 timeout 300 python -m pytest tests/test_tcf_bulk_gpu.py tests/test_acceptance_gpu.py -q -x -k "bulk or c02 or c06 or c07" > gpurun_out/pytest_route.log 2>&1; echo "forced prefix-route pytest rc=$?"; tail -2 gpurun_out/pytest_route.log
timeout 300 python -m pytest tests/test_full_size_gpu.py -q -x -k "bulk" > gpurun_out/pytest_route2.log 2>&1; echo "2^23 pytest rc=$?"; tail -2 gpurun_out/pytest_route2.log
for ls in 24 26; do
  timeout 300 python bench.py --workload bulk_tcf --log-slots $ls --steps 2 --no-cpu --no-e2e --no-launch-count > gpurun_out/br_$ls.json 2>/dev/null
  python -c "
import json
d=json.load(open('gpurun_out/br_$ls.json')); p=d['per_op']; print('$ls', {k:(round(v['ops_per_s']/1e9,3), round(v['ms'],2)) for k,v in p.items()})"
done
