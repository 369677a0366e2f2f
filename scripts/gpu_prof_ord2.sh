#!/usr/bin/env bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_tcf_ordered -c 1 -o gpurun_out/prof_ord_ins -f python scripts/prof_tcf.py 28 ordered > gpurun_out/prof_ord.log 2>&1; echo "ncu ord rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_tcf_insert_cas -c 1 -o gpurun_out/prof_cas_ins -f python scripts/prof_tcf.py 28 concurrent > gpurun_out/prof_cas.log 2>&1; echo "ncu cas rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-concurrent --no-launch-count > gpurun_out/bench_under_ncu.log 2>&1; echo "ncu launches rc=$?"
