#!/usr/bin/env bash
# DRAM bytes / serialised time per kernel of the C4 GQF ops (summaries as r2q_*_dram.json).
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors.sum,lts__t_requests.sum
if [ $# -eq 0 ]; then set -- "gqf_kmer bulk_insert" "gqf_kmer bulk_delete"; fi
for spec in "$@"; do
  set -- $spec
  timeout 900 ncu --profile-from-start off --metrics $M --csv --log-file gpurun_out/d_$1_$2.csv python scripts/prof_workloads.py $1 $2 > gpurun_out/d_$1_$2.out 2>&1
  items=$(python -c "import json;print(json.loads(open('gpurun_out/d_$1_$2.out').read().strip().splitlines()[-1])['items'])")
  python scripts/prof_workloads.py --summarize gpurun_out/d_$1_$2.csv $1 $2 $items gpurun_out/${TAG:-r2q}_$1_$2_dram.json > /dev/null 2>&1; echo "$1 $2 rc=$?"
  rm -f gpurun_out/d_$1_$2.csv
done
