#!/usr/bin/env bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_tcf -c 4 -o gpurun_out/prof_tcf_ordered_d -f python scripts/prof_tcf.py 28 ordered > gpurun_out/prof_d.log 2>&1; echo "ncu full rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_d.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-concurrent --no-launch-count > /dev/null 2>&1; echo "ncu launches rc=$?"
