#!/usr/bin/env bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gqf_gpu.py tests/test_acceptance_gpu.py tests/test_cli.py -m gpu -q -x --durations=8 > gpurun_out/pytest_gqf.log 2>&1; echo "pytest rc=$?"; tail -20 gpurun_out/pytest_gqf.log
