cd "${GRAFT_REPO_ROOT:-.}"
timeout 900 python -m pytest tests/test_tcf_gpu.py -x -q 2>&1 | tail -2
for w in 262144 1048576 4194304; do
  FK_ORD_WINDOW=$w timeout 300 python bench.py --steps 2 --no-cpu --no-e2e --mode ordered | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('W=$w', 'value %.3g'%d['value'], {k:(round(v['ops_per_s']/1e9,2), round(v['ms'],1)) for k,v in d['per_op'].items()})"
done
