#!/usr/bin/env bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -8 gpurun_out/pytest_gpu.log
summ() { python -c "
import json
d=json.load(open('$1')); print('$2 value %.3g'%d['value'], {k:round(v['ops_per_s']/1e9,2) for k,v in d['per_op'].items()}, {k:round(v['ops_per_s']/1e9,2) for k,v in d['concurrent_mode'].items() if isinstance(v,dict)})"; }
timeout 600 python bench.py --steps 3 --no-cpu --no-e2e > gpurun_out/bench_mb5.json 2>/dev/null; summ gpurun_out/bench_mb5.json mb5
cp paper_2212_09005_b200/libfkb200.so /tmp/keep.so; cp build/v6/libfkb200.so paper_2212_09005_b200/libfkb200.so
timeout 600 python bench.py --steps 3 --no-cpu --no-e2e > gpurun_out/bench_mb6.json 2>/dev/null; summ gpurun_out/bench_mb6.json mb6
cp /tmp/keep.so paper_2212_09005_b200/libfkb200.so
