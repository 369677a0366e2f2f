#!/usr/bin/env bash
# Round-2 late: lanes per key of the bulk-TCF query -- parity at G = 2/4, then A/B.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
T=${TAG:-r2q3}
for g in 1 2; do
FK_BTCF_QUERY_G=$g timeout 900 python -m pytest tests/test_tcf_bulk_gpu.py -m gpu -q -x > gpurun_out/${T}_pytest_g$g.log 2>&1; echo "pytest G=$g rc=$?"; tail -1 gpurun_out/${T}_pytest_g$g.log
done
for g in 8 2 1 8 2 1; do
FK_BTCF_QUERY_G=$g timeout 600 python bench.py --workload bulk_tcf --steps 200 --warmup 3 --no-e2e --no-cpu > gpurun_out/${T}_bulk_g$g.json 2>/dev/null
python -c "
import json; b=json.loads(open('gpurun_out/${T}_bulk_g$g.json').read().strip().splitlines()[-1]); print('G=$g', round(b['value']/1e9,3), {k:round(x['ms'],4) for k,x in b['per_op'].items()})"
done
