#!/usr/bin/env bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest_gpu.log
timeout 600 python scripts/ord_tune.py --log-slots 20 22 24 28 --cfg default > gpurun_out/ord_tune3.jsonl 2> gpurun_out/ord_tune3.err; echo "tune rc=$?"
timeout 600 python bench.py --steps 3 --no-cpu --no-e2e > gpurun_out/bench_quick.json 2> gpurun_out/bench_quick.err; echo "bench rc=$?"
python -c "
import json
d=json.load(open('gpurun_out/bench_quick.json')); print('value %.3g'%d['value'], {k:round(v['ops_per_s']/1e9,2) for k,v in d['per_op'].items()}, {k:round(v['ops_per_s']/1e9,2) for k,v in d['concurrent_mode'].items() if isinstance(v,dict)})"
