#!/bin/bash
# round 2: cluster ring — relaxed vs release remote arrives, and wait-time profile
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
export POLAR_TIMEOUT_MS=20000 AB_SIZES_MIB=${AB_SIZES_MIB:-1,8,32,128} AB_VARIANTS="POLAR_CLUSTER=1"
for L in cur clrel; do
  if [ $L = cur ]; then unset POLAR_LIB; else export POLAR_LIB=build/variants/libpolar_$L.so; fi
  timeout 300 python scripts/experiments/exp_ring_tma.py 2> gpurun_out/r02u_$L.err | sed "s/^/$L /" | tee -a gpurun_out/r02u_ab.jsonl | cut -c1-190
  tail -2 gpurun_out/r02u_$L.err
done
POLAR_LIB=build/variants/libpolar_clprof.so timeout 120 python scripts/experiments/exp_cl_prof.py 2>&1 | tee gpurun_out/r02u_prof.jsonl
