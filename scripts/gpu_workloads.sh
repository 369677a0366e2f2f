#!/usr/bin/env bash
# Secondary workloads: bulk TCF and GQF bench lines + ncu launch lists.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
for w in bulk_tcf gqf; do
  timeout 900 python bench.py --workload $w --steps 3 ${EXTRA} > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err; echo "$w rc=$?"
  tail -c 2500 gpurun_out/bench_$w.json; tail -3 gpurun_out/bench_$w.err
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$w.csv python bench.py --workload $w --steps 1 --warmup 3 --no-e2e --no-cpu --no-launch-count > /dev/null 2>&1; echo "ncu $w rc=$?"
done
