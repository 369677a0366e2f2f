#!/usr/bin/env bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
FK_ROUTE_PREFIX=1 timeout 300 python -m pytest tests/test_tcf_bulk_gpu.py tests/test_acceptance_gpu.py -q -x -k "bulk or c02 or c06 or c07" > gpurun_out/pytest_route.log 2>&1; echo "prefix-route pytest rc=$?"; tail -3 gpurun_out/pytest_route.log
for ls in 20 24 26; do for v in warp prefix; do
  if [ $v = warp ]; then export FK_ROUTE_WARP=1; unset FK_ROUTE_PREFIX; else unset FK_ROUTE_WARP; export FK_ROUTE_PREFIX=1; fi
  timeout 300 python bench.py --workload bulk_tcf --log-slots $ls --steps 2 --no-cpu --no-e2e --no-launch-count > gpurun_out/br_${ls}_$v.json 2>/dev/null
  python -c "
import json
d=json.load(open('gpurun_out/br_${ls}_$v.json')); p=d['per_op']; print('$ls $v', {k:(round(v['ops_per_s']/1e9,3), round(v['ms'],2)) for k,v in p.items()})"
done; done
