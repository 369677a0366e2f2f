#!/usr/bin/env bash
# ncu DRAM bytes per item for the secondary workloads' ops (whole-op sums).
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sectors.sum,lts__t_requests.sum
for wo in "bulk_tcf insert" "bulk_tcf query_pos" "gqf bulk_insert" "gqf count" "gqf bulk_delete" "gqf_kmer bulk_insert" "gqf_kmer count" "gqf_kmer bulk_delete"; do
  set -- $wo
  timeout 900 ncu --profile-from-start off --clock-control none --metrics $M --csv --log-file gpurun_out/r2e_$1_$2.csv python scripts/prof_workloads.py $1 $2 > gpurun_out/r2e_$1_$2.out 2>&1; echo "$1 $2 rc=$?"; tail -1 gpurun_out/r2e_$1_$2.out
done
