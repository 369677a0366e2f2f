#!/usr/bin/env bash
# GPU parity tests (optionally a subset: scripts/gpu_tests.sh tests/test_x.py)
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 1500 python -m pytest ${@:-tests} -m gpu -x -q 2>&1 | tail -40 | tee gpurun_out/pytest_gpu.log
