#!/usr/bin/env bash
# Round-2 first check: smoke, GPU tests, headline bench on the current head.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2a_smi.txt 2>&1
lscpu > gpurun_out/r2a_lscpu.txt 2>&1
timeout 240 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r2a_smoke.log 2>&1; echo "smoke rc=$?"
timeout 1200 python -m pytest tests -m gpu -q -x --durations=15 > gpurun_out/r2a_pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -25 gpurun_out/r2a_pytest_gpu.log
timeout 600 python bench.py > gpurun_out/r2a_bench.json 2> gpurun_out/r2a_bench.err; echo "bench rc=$?"; tail -c 600 gpurun_out/r2a_bench.json
