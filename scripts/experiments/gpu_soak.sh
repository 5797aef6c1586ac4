#!/bin/bash
# Soak: the random stress tests with fresh seeds, longer (virtual comms, then 8
# processes under MPS with and without fault delays).
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
POLAR_STRESS_SEED=7 POLAR_STRESS_S=600 POLAR_TIMEOUT_MS=20000 timeout 900 python -m pytest tests/test_gpu_stress.py -x -q -s \
  > gpurun_out/soak_virtual.log 2>&1; echo "virtual rc=$?"; grep -o "stress: [^;]*;" gpurun_out/soak_virtual.log
export POLAR_STRESS_SEED=11 POLAR_STRESS_S=300
bash scripts/experiments/gpu_mps_stress.sh
