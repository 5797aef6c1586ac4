#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
export POLAR_TIMEOUT_MS=5000
timeout 300 python scripts/probe_ll128.py > gpurun_out/probe_ll128.jsonl 2>&1; echo "probe rc=$?"; cat gpurun_out/probe_ll128.jsonl
timeout 600 python -m pytest tests/test_gpu_faults.py tests/test_gpu_multiproc.py -q -x --timeout=300 > gpurun_out/pytest_faults.log 2>&1
echo "faults rc=$?"; tail -3 gpurun_out/pytest_faults.log
