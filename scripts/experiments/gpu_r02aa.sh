#!/bin/bash
# cluster tree: parity, A/B vs the FIFO tree
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
export POLAR_TIMEOUT_MS=5000
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "tree and simple" 2>&1 | tail -4
export POLAR_TIMEOUT_MS=20000 AB_SIZES_MIB=${AB_SIZES_MIB:-1,8,32,128} AB_ALGOS=tree
AB_VARIANTS="POLAR_CLUSTER=0,POLAR_CLUSTER=1" timeout 300 python scripts/experiments/exp_ring_tma.py 2> gpurun_out/r02aa.err | tee gpurun_out/r02aa_ab.jsonl | cut -c1-175
tail -2 gpurun_out/r02aa.err
