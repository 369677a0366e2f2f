#!/usr/bin/env bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_gqf_kmer.csv python bench.py --workload gqf_kmer --steps 1 --warmup 3 --no-e2e --no-cpu --no-launch-count > /dev/null 2>&1; echo "ncu gqf rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-concurrent --no-launch-count > /dev/null 2>&1; echo "ncu launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_tcf -c 4 -o gpurun_out/prof_tcf_ordered_c -f python scripts/prof_tcf.py 28 ordered > gpurun_out/prof_c.log 2>&1; echo "ncu full rc=$?"
