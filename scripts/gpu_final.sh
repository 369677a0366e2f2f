#!/usr/bin/env bash
# Round-end evidence: smoke, GPU tests, every bench line, ncu of the C3 kernels.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 240 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo "bench rc=$?"
for w in bulk_tcf gqf gqf_kmer; do timeout 600 python bench.py --workload $w --steps 3 > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err; echo "$w rc=$?"; done
timeout 600 python bench.py --impl reference --steps 2 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_tcf -c 4 -o gpurun_out/prof_tcf_f -f python scripts/prof_tcf.py 28 ordered > gpurun_out/prof_f.log 2>&1; echo "ncu full rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_f.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-concurrent --no-launch-count > /dev/null 2>&1; echo "ncu launches rc=$?"
