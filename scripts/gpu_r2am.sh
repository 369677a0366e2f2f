#!/usr/bin/env bash
# Round-2 late: warp-merged partition aggregation (GQF) -- parity, then A/B on C4 / C2.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
T=${TAG:-r2am}
timeout 1200 python -m pytest tests/test_gqf_gpu.py tests/test_full_size_gpu.py -m gpu -q -x -k "gqf or c2 or c4" > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/${T}_pytest.log
for v in 0 1 0 1; do for w in gqf_kmer gqf; do
FK_GQF_AGG_MATCH=$v timeout 600 python bench.py --workload $w --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/${T}_${w}_$v.json 2>/dev/null
python -c "
import json; b=json.loads(open('gpurun_out/${T}_${w}_$v.json').read().strip().splitlines()[-1]); print('$w match=$v', round(b['value']/1e9,3), {k:round(x['ms'],3) for k,x in b['per_op'].items()})"
done; done
