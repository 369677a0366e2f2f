#!/usr/bin/env bash
# Full-size bit-exact tests (C3 2^28 ordered, C2 q=22, C4 q=28) + the GQF capacity tests.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
free -g > gpurun_out/r2b_free.txt
timeout 2400 python -m pytest tests/test_full_size_gpu.py tests/test_gqf_gpu.py -m gpu -q -x --durations=10 > gpurun_out/r2b_pytest.log 2>&1; echo "pytest rc=$?"; tail -30 gpurun_out/r2b_pytest.log
