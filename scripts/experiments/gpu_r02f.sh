#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
export POLAR_TIMEOUT_MS=20000
timeout 2400 python -m pytest tests -m gpu -q -rs --timeout=900 > gpurun_out/r02f_pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -8 gpurun_out/r02f_pytest_gpu.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/r02f_smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/r02f_smoke.log
