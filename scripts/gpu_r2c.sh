#!/usr/bin/env bash
# Router modes + contract module + reference suite; bulk TCF bench with route stats.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_tcf_bulk_gpu.py -m gpu -q -x > gpurun_out/r2c_bulk.log 2>&1; echo "bulk rc=$?"; tail -3 gpurun_out/r2c_bulk.log
FK_ROUTE_STATS=1 timeout 600 python bench.py --workload bulk_tcf --steps 5 --no-cpu > gpurun_out/r2c_bench_bulk.json 2> gpurun_out/r2c_bench_bulk.err; echo "bench bulk rc=$?"; grep "fk route" gpurun_out/r2c_bench_bulk.err | sort | uniq -c | head -5; tail -c 1500 gpurun_out/r2c_bench_bulk.json
for ls in 22 24; do FK_ROUTE_STATS=1 timeout 600 python bench.py --workload bulk_tcf --log-slots $ls --steps 3 --no-cpu --no-e2e > gpurun_out/r2c_bench_bulk_$ls.json 2> gpurun_out/r2c_bench_bulk_$ls.err; echo "bench bulk $ls rc=$?"; grep "fk route" gpurun_out/r2c_bench_bulk_$ls.err | head -2; done
timeout 2400 python -m pytest tests/test_reference_suite_gpu.py -m gpu -q -x > gpurun_out/r2c_refsuite.log 2>&1; echo "refsuite rc=$?"; tail -40 gpurun_out/r2c_refsuite.log
