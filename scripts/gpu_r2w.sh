#!/usr/bin/env bash
# Round-2 late: count-routed commit of the one-barrier ordered insert --
# ordered parity tests, then A/B against the block-reading commit.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
T=${1:-r2w}
timeout 600 python -m pytest tests/test_tcf_gpu.py -m gpu -q -x -k "ordered" > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/${T}_pytest.log
timeout 600 python scripts/ord_tune.py --log-slots ${LOGS:-24 28} --cfg ${CFGS:-LC=0 LC=1 LC=0 LC=1} > gpurun_out/${T}_ord_tune.jsonl 2>&1; echo "tune rc=$?"
python - gpurun_out/${T}_ord_tune.jsonl <<'PY'
import json,sys
for l in open(sys.argv[1]):
    try: d=json.loads(l)
    except Exception: print(l[:300]); continue
    print(d["log_slots"], d["cfg"], "ins %.3f ms" % d["insert"]["ms"], "del %.3f ms" % d["delete"]["ms"])
PY
