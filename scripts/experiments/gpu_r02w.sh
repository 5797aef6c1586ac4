#!/bin/bash
# round 2: cluster ring v2 (signal warp, receiver-armed full) — parity, A/B vs FIFO ring, wait profile
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
export POLAR_TIMEOUT_MS=5000
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "ring and simple" 2>&1 | tail -3
export POLAR_TIMEOUT_MS=20000 AB_SIZES_MIB=${AB_SIZES_MIB:-1,8,32,128} AB_VARIANTS="POLAR_CLUSTER=1"
timeout 300 python scripts/experiments/exp_ring_tma.py 2> gpurun_out/r02w.err | tee gpurun_out/r02w_ab.jsonl | cut -c1-190
tail -2 gpurun_out/r02w.err
POLAR_LIB=build/variants/libpolar_clprof.so timeout 120 python scripts/experiments/exp_cl_prof.py 2>&1 | tee gpurun_out/r02w_prof.jsonl
