#!/bin/bash
# A/B of build variants (build/variants/libpolar_<name>.so) on the cluster ring / tree:
#   bash scripts/experiments/gpu_lib_ab.sh <tag> cur name1 name2 ...   (AB_ALGOS, AB_SIZES_MIB, AB_DTYPES as in exp_ring_tma.py)
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
TAG=$1; shift
export POLAR_TIMEOUT_MS=${POLAR_TIMEOUT_MS:-5000}
export AB_VARIANTS=${AB_VARIANTS:-POLAR_CLUSTER=1}
export AB_ALGOS=${AB_ALGOS:-ring} AB_SIZES_MIB=${AB_SIZES_MIB:-8,32,128} AB_DTYPES=${AB_DTYPES:-f32,bf16}
for rep in 1 2; do
  for L in "$@"; do
    if [ $L = cur ]; then unset POLAR_LIB; else export POLAR_LIB=build/variants/libpolar_$L.so; fi
    timeout 300 python scripts/experiments/exp_ring_tma.py 2>gpurun_out/ab_${TAG}_$L.err | sed "s/^/$L /" >> gpurun_out/ab_$TAG.jsonl
    echo "$L rc=${PIPESTATUS[0]}" >> gpurun_out/ab_$TAG.jsonl
  done
done
