cd "${GRAFT_REPO_ROOT:-.}"
FK_ORD_WINDOW=262144 ncu --set full --import-source on --clock-control none -k regex:k_tcf_ordered -c 1 -o gpurun_out/prof_ord python scripts/prof_tcf.py 28 ordered > gpurun_out/prof_ord.log 2>&1
tail -3 gpurun_out/prof_ord.log
