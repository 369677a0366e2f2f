#!/usr/bin/env bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gqf_gpu.py tests/test_acceptance_gpu.py tests/test_sharding_gpu.py -q -x > gpurun_out/pytest_gqf.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gqf.log
timeout 900 python bench.py --workload gqf_kmer --steps 3 --no-cpu --no-e2e > gpurun_out/bench_gqf_kmer3.json 2>/dev/null; python -c "
import json
d=json.load(open('gpurun_out/bench_gqf_kmer3.json')); print('gqf_kmer value %.3g'%d['value'], {k:(round(v['ops_per_s']/1e9,2), round(v['ms'],1)) for k,v in d['per_op'].items()})"
