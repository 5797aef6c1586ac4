#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
export POLAR_TIMEOUT_MS=20000 AB_SIZES_MIB=${AB_SIZES_MIB:-1,8,32,128}
AB_VARIANTS="POLAR_RING_STAGE=0,POLAR_RING_STAGE=1" timeout 900 python scripts/experiments/exp_ring_tma.py > gpurun_out/r02n_ab.jsonl 2> gpurun_out/r02n_ab.err; echo "ab rc=$?"
cut -c1-175 gpurun_out/r02n_ab.jsonl; tail -3 gpurun_out/r02n_ab.err
