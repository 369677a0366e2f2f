#!/usr/bin/env bash
# One GPU call: parity tests + bench line (+ optional ncu passes: PROF=1).
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -5 gpurun_out/pytest_gpu.log
timeout 900 python bench.py ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
tail -c 4000 gpurun_out/bench.json; tail -5 gpurun_out/bench.err
if [ -n "$PROF" ]; then
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-concurrent --no-launch-count > gpurun_out/bench_under_ncu.log 2>&1; echo "ncu1 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_tcf -c 4 -o gpurun_out/prof_tcf_ordered -f python scripts/prof_tcf.py 28 ordered > gpurun_out/prof1.log 2>&1; echo "ncu2 rc=$?"
fi
