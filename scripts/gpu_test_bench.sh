cd "${GRAFT_REPO_ROOT:-.}"
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
for m in ordered concurrent; do
  timeout 300 python bench.py --steps 3 --no-cpu --no-e2e --mode $m | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print(d['config']['mode'], 'value %.3g'%d['value'], {k:(round(v['ops_per_s']/1e9,2), round(v['achieved_gbs'])) for k,v in d['per_op'].items()}, d['checks'])"
done
