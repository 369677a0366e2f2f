#!/usr/bin/env bash
# Round-2 late: wider ordered window (4 keys per thread at 3 CTAs/SM) A/B.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
T=${TAG:-r2v}
FK_ORD_WIDE=1 timeout 600 python -m pytest tests/test_tcf_gpu.py -m gpu -q -x -k "ordered" > gpurun_out/${T}_pytest.log 2>&1; echo "pytest(wide) rc=$?"; tail -2 gpurun_out/${T}_pytest.log
timeout 900 python scripts/ord_tune.py --log-slots 24 28 --cfg WIDE=0 WIDE=1 WIDE=1,W=350000 WIDE=1,W=524288 WIDE=0 WIDE=1,W=524288 > gpurun_out/${T}_ord_tune.jsonl 2>&1; echo "tune rc=$?"
python - gpurun_out/${T}_ord_tune.jsonl <<'PY'
import json,sys
for l in open(sys.argv[1]):
    try: d=json.loads(l)
    except Exception: print(l[:300]); continue
    print(d["log_slots"], d["cfg"], "ins %.3f ms rounds %d carried %d" % (d["insert"]["ms"], d["insert"]["rounds"], d["insert"]["carried"]), "del %.3f ms" % d["delete"]["ms"])
PY
