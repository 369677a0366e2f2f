#!/usr/bin/env bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:route_jacobi -c 1 -o gpurun_out/r2g_route -f python scripts/prof_workloads.py bulk_tcf insert > gpurun_out/r2g.log 2>&1; echo "ncu rc=$?"; tail -3 gpurun_out/r2g.log
