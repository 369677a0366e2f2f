#!/usr/bin/env bash
# Round-2 late: GQF per-CTA sums (region summary, stats) -- parity and the C2/C4 lines.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
T=${TAG:-r2g2}
timeout 1200 python -m pytest tests/test_gqf_gpu.py tests/test_full_size_gpu.py tests/test_tcf_bulk_gpu.py -m gpu -q -x -k "gqf or c2 or c4 or bulk" > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/${T}_pytest.log
for w in gqf_kmer gqf gqf_kmer gqf; do
timeout 600 python bench.py --workload $w --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/${T}_$w.json 2>/dev/null
python -c "
import json; b=json.loads(open('gpurun_out/${T}_$w.json').read().strip().splitlines()[-1]); print('$w', round(b['value']/1e9,3), {k:round(x['ms'],3) for k,x in b['per_op'].items()})"
done
