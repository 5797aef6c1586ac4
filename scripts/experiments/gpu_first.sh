#!/bin/bash
# first GPU session: smoke, parity tests, a quick sweep
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
export POLAR_TIMEOUT_MS=5000
nvidia-smi > gpurun_out/nvsmi.txt 2>&1
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -q -rf --timeout=400 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python scripts/sweep.py --n 8 --dtype f32 --sizes 4K,64K,1M,4M,32M,128M --nch 4,16,32 > gpurun_out/sweep1.jsonl 2>&1; echo "sweep rc=$?" >> gpurun_out/sweep1.jsonl
tail -3 gpurun_out/smoke.log gpurun_out/pytest_gpu.log
