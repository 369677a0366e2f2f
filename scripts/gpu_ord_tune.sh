#!/usr/bin/env bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_tcf_gpu.py -x -q 2>&1 | tail -2
timeout 600 python scripts/ord_tune.py --log-slots 20 22 --cfg default "RS=0,W=16384" "RS=0,W=131072" "CTAS=2" > gpurun_out/ord_tune_small.jsonl 2> gpurun_out/ord_tune_small.err; echo "small rc=$?"
timeout 900 python scripts/ord_tune.py --log-slots 24 28 --cfg default "CTAS=2" "CTAS=3" "W=131072" "RS=1,W=262144" > gpurun_out/ord_tune_big.jsonl 2> gpurun_out/ord_tune_big.err; echo "big rc=$?"
tail -n 3 gpurun_out/ord_tune_small.err gpurun_out/ord_tune_big.err
