#!/bin/bash
# cluster tree variants (double tree warp groups / stages; single tree)
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
export POLAR_TIMEOUT_MS=20000 AB_SIZES_MIB=${AB_SIZES_MIB:-1,8,32,128} AB_ALGOS=tree AB_DTYPES=f32,bf16 AB_VARIANTS="POLAR_CLUSTER=1;POLAR_CLUSTER_TREE_MAX=1099511627776"
for L in ${VARS:-cur trdsmem}; do
  if [ $L = cur ]; then unset POLAR_LIB; else export POLAR_LIB=build/variants/libpolar_$L.so; fi
  timeout 300 python scripts/experiments/exp_ring_tma.py 2> gpurun_out/r02ee_$L.err | sed "s/^/$L /" | tee -a gpurun_out/r02ee_ab.jsonl | cut -c1-30,130-230
  tail -n 2 gpurun_out/r02ee_$L.err
done
