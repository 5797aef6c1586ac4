#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
export POLAR_TIMEOUT_MS=5000 POLAR_LIB=build/variants/libpolar_cf3.so
for j in 0 3000 20000; do
  for cfg in "8 f32 sum 680 1" "8 i64 min 682 1" "8 f32 sum 4096 1" "8 f32 sum 680 4" "7 f32 sum 680 2" "6 bf16 sum 1000 1" "8 f32 sum 1048576 3"; do
    set -- $cfg
    POLAR_JITTER_NS=$j timeout 60 python scripts/experiments/repro_ulf.py $1 $2 $3 ring $4 $5 100 2>&1 | grep -E "^(OK|FAIL)" | cut -c1-90 | sed "s/^/jit=$j /"
  done
done
POLAR_STRESS_S=240 POLAR_TIMEOUT_MS=20000 timeout 600 python -m pytest tests/test_gpu_stress.py tests/test_gpu_cluster.py -x -q -s 2>&1 | grep -E "stress:|passed|failed" | cut -c1-200
unset POLAR_LIB
AB_SIZES_MIB=8,32,128 bash scripts/experiments/gpu_lib_ab.sh cf3ab cf0 cf3
