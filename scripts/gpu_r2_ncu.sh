#!/usr/bin/env bash
# Round-2 ncu evidence: --set full captures of the C3 point-TCF kernels, the
# C4 GQF insert kernels and the configs[0] bulk-TCF route kernel.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_tcf -c 4 -o gpurun_out/r2_tcf_c3 -f python scripts/prof_tcf.py 28 ordered > gpurun_out/r2_ncu_tcf.log 2>&1; echo "tcf rc=$?"
timeout 1200 ncu --set full --clock-control none --profile-from-start off -k regex:"k_part|k_region" -o gpurun_out/r2_gqf_c4 -f python scripts/prof_workloads.py gqf_kmer bulk_insert > gpurun_out/r2_ncu_gqf.log 2>&1; echo "gqf rc=$?"
timeout 900 ncu --set full --clock-control none --profile-from-start off -k regex:"k_btcf_route_jacobi" -c 1 -o gpurun_out/r2_btcf_route -f python scripts/prof_workloads.py bulk_tcf insert > gpurun_out/r2_ncu_btcf.log 2>&1; echo "btcf rc=$?"
# summaries only (the reports exceed what gpurun brings back)
for r in r2_tcf_c3 r2_gqf_c4 r2_btcf_route; do
  python scripts/ncu_summary.py full gpurun_out/$r.ncu-rep gpurun_out/${r}_full.json > gpurun_out/${r}_summary.log 2>&1; echo "$r summary rc=$?"
  ncu -i gpurun_out/$r.ncu-rep --page raw --csv > gpurun_out/${r}_raw.csv 2>/dev/null
  gzip -f gpurun_out/${r}_raw.csv
  rm -f gpurun_out/$r.ncu-rep
done
ls -la gpurun_out | head -30
