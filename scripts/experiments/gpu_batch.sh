#!/bin/bash
# full GPU suite + protocol sweep + bench (round-1 batching work)
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
TAG=${1:-r01f}
export POLAR_TIMEOUT_MS=5000
timeout 1500 python -m pytest tests -m gpu -q -rf --timeout=600 > gpurun_out/pytest_gpu_$TAG.log 2>&1
echo "pytest rc=$?"; tail -6 gpurun_out/pytest_gpu_$TAG.log
timeout 900 python scripts/sweep.py --n 8 --dtype f32 --sizes 64K,1M,4M,16M,32M,128M \
  --algos oneshot:ll,oneshot:ll128,oneshot:simple,twoshot:ll,twoshot:ll128,twoshot:simple,ring:ll,ring:ll128,ring:simple,tree:ll,tree:ll128,tree:simple \
  --nch 4,8,16,32 > gpurun_out/sweep_$TAG.jsonl 2>&1
echo "sweep rc=$?"
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
echo "bench rc=$?"; cut -c1-400 gpurun_out/bench_$TAG.json
