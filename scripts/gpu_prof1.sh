cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench_under_ncu.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_tcf -c 4 -o gpurun_out/prof_tcf_ordered python scripts/prof_tcf.py 28 ordered > gpurun_out/prof1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_tcf_insert_cas -c 1 -o gpurun_out/prof_tcf_cas python scripts/prof_tcf.py 28 concurrent > gpurun_out/prof2.log 2>&1
ls -la gpurun_out
