#!/usr/bin/env bash
# Round-2 late: L2-blocked batch query -- parity tests, then A/B on the C3 bench line.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
T=${TAG:-r2y}
timeout 900 python -m pytest tests/test_tcf_gpu.py tests/test_full_size_gpu.py -m gpu -q -x -k "blocked or query or ordered_2p24 or c3_2p28_ordered or golden or c1" > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/${T}_pytest.log
for cl in 25 24 26; do
FK_QBLOCK_CHUNK_LOG=$cl timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --no-concurrent --no-secondary > gpurun_out/${T}_bench_cl$cl.json 2> gpurun_out/${T}_bench_cl$cl.err; echo "bench cl=$cl rc=$?"
done
FK_QBLOCK=0 timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --no-concurrent --no-secondary > gpurun_out/${T}_bench_off.json 2> gpurun_out/${T}_bench_off.err; echo "bench off rc=$?"
python - <<'PY'
import json,glob
for f in sorted(glob.glob("gpurun_out/r2y_bench_*.json")):
    try:
        b=json.loads(open(f).read().strip().splitlines()[-1])
        print(f, round(b["value"]/1e9,2), {k:round(v["ms"],2) for k,v in b["per_op"].items()})
    except Exception as e: print(f, "ERR", e)
PY
