#!/usr/bin/env bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_tcf_gpu.py -x -q -k "pipeline or c1_full" > gpurun_out/pytest_pipe.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/pytest_pipe.log
timeout 900 python bench.py --steps 3 --no-cpu --no-concurrent > gpurun_out/bench_e2e.json 2>gpurun_out/bench_e2e.err; echo "bench rc=$?"; tail -3 gpurun_out/bench_e2e.err; python -c "
import json
d=json.load(open('gpurun_out/bench_e2e.json')); print('value %.3g'%d['value'], 'e2e', d['e2e'])"
