#!/usr/bin/env bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gqf_gpu.py tests/test_acceptance_gpu.py tests/test_cli.py tests/test_sharding_gpu.py -q -x > gpurun_out/pytest_gqf.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gqf.log
