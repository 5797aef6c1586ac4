#!/bin/bash
# round 2: cluster-transport ring (cluster.cuh) — parity, then A/B against the FIFO ring
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
export POLAR_TIMEOUT_MS=5000
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "ring and simple" 2>&1 | tail -15; echo "pytest rc=$?"
export POLAR_TIMEOUT_MS=20000 AB_SIZES_MIB=${AB_SIZES_MIB:-1,8,32,128}
AB_VARIANTS="POLAR_CLUSTER=0,POLAR_CLUSTER=1" timeout 600 python scripts/experiments/exp_ring_tma.py > gpurun_out/r02s_ab.jsonl 2> gpurun_out/r02s_ab.err; echo "ab rc=$?"
cut -c1-200 gpurun_out/r02s_ab.jsonl; tail -3 gpurun_out/r02s_ab.err
