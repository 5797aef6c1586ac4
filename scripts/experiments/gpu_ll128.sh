#!/bin/bash
# LL128 bring-up: full GPU suite + protocol sweep on 8 virtual ranks
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
export POLAR_TIMEOUT_MS=5000
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "ll128" --timeout=300 > gpurun_out/pytest_ll128.log 2>&1
echo "ll128 pytest rc=$?"; tail -5 gpurun_out/pytest_ll128.log
timeout 1500 python -m pytest tests -m gpu -q -rf --timeout=600 > gpurun_out/pytest_gpu_all.log 2>&1
echo "all pytest rc=$?"; tail -5 gpurun_out/pytest_gpu_all.log
timeout 600 python scripts/sweep.py --n 8 --dtype f32 --sizes 64K,1M,4M,8M,16M,32M,128M \
  --algos ring:ll,ring:ll128,ring:simple,twoshot:ll,twoshot:ll128,oneshot:ll,oneshot:ll128,tree:ll128,tree:simple \
  --nch 4,8,16,32 > gpurun_out/sweep_ll128.jsonl 2>&1
echo "sweep rc=$?"
