#!/usr/bin/env bash
# Round-2 late: ordered tests + tuning probe on the current head, the default
# bench line, the launch list and an ncu --set full capture of the C3 kernels.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
T=${TAG:-r2x}
timeout 900 python -m pytest tests/test_tcf_gpu.py tests/test_full_size_gpu.py -m gpu -q -x -k "ordered or c3 or concurrent or cas" > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/${T}_pytest.log
timeout 600 python scripts/ord_tune.py --log-slots 20 22 24 28 > gpurun_out/${T}_ord_tune.jsonl 2>&1; echo "tune rc=$?"
timeout 900 python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err; echo "bench rc=$?"; tail -2 gpurun_out/${T}_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-concurrent --no-launch-count --no-secondary > /dev/null 2>&1; echo "ncu launches rc=$?"
python scripts/ncu_summary.py launches gpurun_out/${T}_launches.csv gpurun_out/${T}_launches.json > /dev/null 2>&1; echo "summary rc=$?"
rm -f gpurun_out/${T}_launches.csv
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_tcf -c 4 -o gpurun_out/${T}_tcf_c3 -f python scripts/prof_tcf.py 28 ordered > gpurun_out/${T}_ncu_tcf.log 2>&1; echo "tcf ncu rc=$?"
python scripts/ncu_summary.py full gpurun_out/${T}_tcf_c3.ncu-rep gpurun_out/${T}_tcf_point_ordered_full.json > gpurun_out/${T}_tcf_summary.log 2>&1; echo "summary rc=$?"
ncu -i gpurun_out/${T}_tcf_c3.ncu-rep --page raw --csv > gpurun_out/${T}_tcf_c3_raw.csv 2>/dev/null; gzip -f gpurun_out/${T}_tcf_c3_raw.csv
rm -f gpurun_out/${T}_tcf_c3.ncu-rep
