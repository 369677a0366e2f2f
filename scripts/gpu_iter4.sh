#!/usr/bin/env bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/pytest_gpu.log
for pf in 0 1; do FK_ORD_PREFETCH=$pf timeout 600 python scripts/ord_tune.py --log-slots 22 24 28 --cfg default > gpurun_out/ord_tune_pf$pf.jsonl 2>/dev/null; echo "pf=$pf"; python -c "
import json
for l in open('gpurun_out/ord_tune_pf$pf.jsonl'):
    d=json.loads(l); print(d['log_slots'], *['%s %.2fG/s us/r=%.1f'%(op[:3],d[op]['g_ops_per_s'],d[op]['us_per_round']) for op in ('insert','delete')])"; done
timeout 900 python bench.py --workload gqf_kmer --steps 3 --no-cpu --no-e2e > gpurun_out/bench_gqf_kmer2.json 2>/dev/null; python -c "
import json
d=json.load(open('gpurun_out/bench_gqf_kmer2.json')); print('gqf_kmer value %.3g'%d['value'], {k:(round(v['ops_per_s']/1e9,2), round(v['ms'],1)) for k,v in d['per_op'].items()})"
timeout 600 python bench.py --steps 3 --no-cpu --no-e2e > gpurun_out/bench_quick.json 2>/dev/null; python -c "
import json
d=json.load(open('gpurun_out/bench_quick.json')); print('value %.3g'%d['value'], {k:round(v['ops_per_s']/1e9,2) for k,v in d['per_op'].items()}, {k:round(v['ops_per_s']/1e9,2) for k,v in d['concurrent_mode'].items() if isinstance(v,dict)})"
