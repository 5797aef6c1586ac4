#!/bin/bash
# unregistered two-shot: own shard direct (default) vs full bounce — multi-process tests + MPS bench N = 2, 4
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
export POLAR_TIMEOUT_MS=20000
timeout 1200 python -m pytest tests/test_gpu_multiproc.py tests/test_gpu_bench.py -x -q > gpurun_out/r02jj_tests.log 2>&1; tail -2 gpurun_out/r02jj_tests.log
TAG=_own bash scripts/gpu_mps_bench.sh 2 4
TAG=_full POLAR_BOUNCE_FULL=1 bash scripts/gpu_mps_bench.sh 2 4
