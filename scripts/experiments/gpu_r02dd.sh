#!/bin/bash
# cluster tree as a double binary tree: tests, A/B vs the FIFO tree
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
export POLAR_TIMEOUT_MS=10000
timeout 900 python -m pytest tests/test_gpu_cluster.py -x -q > gpurun_out/r02dd_test.log 2>&1; tail -3 gpurun_out/r02dd_test.log
export POLAR_TIMEOUT_MS=20000 AB_SIZES_MIB=${AB_SIZES_MIB:-1,8,32,128} AB_ALGOS=tree
AB_VARIANTS="POLAR_CLUSTER=0,POLAR_CLUSTER=1;POLAR_CLUSTER_TREE_MAX=1099511627776" timeout 300 python scripts/experiments/exp_ring_tma.py 2> gpurun_out/r02dd.err | tee gpurun_out/r02dd_ab.jsonl | cut -c1-175
tail -2 gpurun_out/r02dd.err
