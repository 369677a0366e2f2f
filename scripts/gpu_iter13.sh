#!/usr/bin/env bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gqf_gpu.py tests/test_acceptance_gpu.py tests/test_cli.py tests/test_sharding_gpu.py -q -x > gpurun_out/pytest_gqf.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gqf.log
for w in gqf gqf_kmer; do timeout 300 python bench.py --workload $w --steps 3 --no-cpu --no-e2e > gpurun_out/b_$w.json 2>/dev/null; python -c "
import json
d=json.load(open('gpurun_out/b_$w.json')); print('$w value %.3g'%d['value'], {k:(round(v['ops_per_s']/1e9,2), round(v['ms'],2)) for k,v in d['per_op'].items()})"; done
