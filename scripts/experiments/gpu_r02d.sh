#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
export POLAR_TIMEOUT_MS=10000
AB_VARIANTS="POLAR_RING_TMA=0,POLAR_RING_TMA_FLAGS=0,POLAR_RING_TMA_FLAGS=1,POLAR_RING_TMA_FLAGS=2,POLAR_RING_TMA_FLAGS=3" AB_SIZES_MIB=8,128 \
  timeout 600 python scripts/experiments/exp_ring_tma.py > gpurun_out/r02d_ring_tma_ab.jsonl 2> gpurun_out/r02d_ring_tma_ab.err; echo "ab rc=$?"
cut -c1-200 gpurun_out/r02d_ring_tma_ab.jsonl; tail -3 gpurun_out/r02d_ring_tma_ab.err
