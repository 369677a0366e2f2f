#!/usr/bin/env bash
# DRAM bytes per op of every secondary workload's op (the bench lines' roofline traffic).
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors.sum,lts__t_requests.sum
for spec in "gqf bulk_insert" "gqf count" "gqf bulk_delete" "gqf_kmer bulk_insert" "gqf_kmer count" "gqf_kmer bulk_delete" "bulk_tcf insert" "bulk_tcf query_pos" "bulk_tcf delete"; do
  set -- $spec
  timeout 900 ncu --profile-from-start off --metrics $M --csv --log-file gpurun_out/d_$1_$2.csv python scripts/prof_workloads.py $1 $2 > gpurun_out/d_$1_$2.out 2>&1
  items=$(python -c "import json;print(json.loads(open('gpurun_out/d_$1_$2.out').read().strip().splitlines()[-1])['items'])")
  python scripts/prof_workloads.py --summarize gpurun_out/d_$1_$2.csv $1 $2 $items gpurun_out/r2p_$1_$2_dram.json > /dev/null 2>&1; echo "$1 $2 rc=$?"
  rm -f gpurun_out/d_$1_$2.csv
done
