#!/usr/bin/env bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_tcf_bulk_gpu.py tests/test_full_size_gpu.py -k "bulk or route" -m gpu -q -x > gpurun_out/r2f_bulk.log 2>&1; echo "bulk rc=$?"; tail -3 gpurun_out/r2f_bulk.log
for ls in 20 22 24; do FK_ROUTE_STATS=1 timeout 600 python bench.py --workload bulk_tcf --log-slots $ls --steps 3 --no-cpu --no-e2e --exact-steps > gpurun_out/r2f_bench_bulk_$ls.json 2> gpurun_out/r2f_bench_bulk_$ls.err; echo "bench bulk $ls rc=$?"; grep "fk route" gpurun_out/r2f_bench_bulk_$ls.err | head -1; python -c "
import json;d=json.loads(open('gpurun_out/r2f_bench_bulk_$ls.json').read().strip().splitlines()[-1]);print({k:round(v['ms'],3) for k,v in d['per_op'].items()}, d['value']/1e9)"; done
timeout 600 ncu --profile-from-start off --clock-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv --log-file gpurun_out/r2f_bulk_tcf_insert.csv python scripts/prof_workloads.py bulk_tcf insert > /dev/null 2>&1; echo "ncu rc=$?"
