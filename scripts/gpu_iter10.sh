#!/usr/bin/env bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gqf_gpu.py tests/test_acceptance_gpu.py tests/test_cli.py -q -x > gpurun_out/pytest_gqf.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gqf.log
timeout 300 python scripts/gqf_small_batch.py 28 > gpurun_out/gqf_small.jsonl 2> gpurun_out/gqf_small.err; echo "small rc=$?"; cat gpurun_out/gqf_small.jsonl; tail -3 gpurun_out/gqf_small.err
