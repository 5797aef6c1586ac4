#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
export POLAR_TIMEOUT_MS=10000
export AB_SIZES_MIB=8,128
AB_VARIANTS="POLAR_RING_TMA=0,POLAR_RING_TMA_FLAGS=0,POLAR_RING_TMA_FLAGS=1" timeout 600 python scripts/experiments/exp_ring_tma.py > gpurun_out/r02e_ab.jsonl 2> gpurun_out/r02e_ab.err; echo "ab rc=$?"
POLAR_LIB=$PWD/build/variants/libpolar_t1024.so AB_VARIANTS="POLAR_RING_TMA_FLAGS=0;T=1024,POLAR_RING_TMA_FLAGS=1;T=1024" timeout 600 python scripts/experiments/exp_ring_tma.py >> gpurun_out/r02e_ab.jsonl 2>> gpurun_out/r02e_ab.err; echo "ab2 rc=$?"
cut -c1-170 gpurun_out/r02e_ab.jsonl; tail -3 gpurun_out/r02e_ab.err
