#!/usr/bin/env bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 2400 python -m pytest tests/test_reference_suite_gpu.py -m gpu -q > gpurun_out/r2d_refsuite.log 2>&1; echo "refsuite rc=$?"; tail -5 gpurun_out/r2d_refsuite.log
for f in gpurun_out/refsuite_*.log; do echo "== $f"; grep -E "^(FAILED|ERROR)|passed|failed" $f | tail -30; done
