#!/bin/bash
# cluster ring v4 (all-gather through L2): parity, A/B vs v3 (all-gather over DSMEM)
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
export POLAR_TIMEOUT_MS=5000
timeout 600 python -m pytest tests/test_gpu_cluster.py -x -q -k "ring or dispatch or graph or jitter" > gpurun_out/r02cc_test.log 2>&1; tail -3 gpurun_out/r02cc_test.log
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "ring and simple" 2>&1 | tail -2
export POLAR_TIMEOUT_MS=20000 AB_SIZES_MIB=${AB_SIZES_MIB:-1,8,32,128} AB_VARIANTS="POLAR_CLUSTER=1"
for L in ${VARS:-cur v3}; do
  if [ $L = cur ]; then unset POLAR_LIB; else export POLAR_LIB=build/variants/libpolar_$L.so; fi
  timeout 300 python scripts/experiments/exp_ring_tma.py 2> gpurun_out/r02cc_$L.err | sed "s/^/$L /" | tee -a gpurun_out/r02cc_ab.jsonl | cut -c1-175
  tail -2 gpurun_out/r02cc_$L.err
done
