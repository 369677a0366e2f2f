#!/usr/bin/env bash
# C3 CG sweep + C4 GQF load sweep + C4 bench line (one GPU call).
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 300 python scripts/gqf_load_sweep.py --q 22 --alphas 0.5 0.9 > gpurun_out/gqf_sweep_q22.jsonl 2> gpurun_out/gqf_sweep_q22.err; echo "sweep22 rc=$?"
tail -3 gpurun_out/gqf_sweep_q22.err
timeout 1200 python scripts/gqf_load_sweep.py --q 28 > gpurun_out/gqf_sweep_q28.jsonl 2> gpurun_out/gqf_sweep_q28.err; echo "sweep28 rc=$?"
tail -3 gpurun_out/gqf_sweep_q28.err
timeout 900 python bench.py --workload gqf_kmer --steps 3 > gpurun_out/bench_gqf_kmer.json 2> gpurun_out/bench_gqf_kmer.err; echo "bench kmer rc=$?"
tail -3 gpurun_out/bench_gqf_kmer.err
timeout 1200 python scripts/cg_sweep.py > gpurun_out/cg_sweep.jsonl 2> gpurun_out/cg_sweep.err; echo "cg rc=$?"
tail -3 gpurun_out/cg_sweep.err
