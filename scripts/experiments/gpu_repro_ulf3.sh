#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
export POLAR_TIMEOUT_MS=5000
for j in 0 3000 20000; do
  for cfg in "8 f32 sum 680 1" "8 i64 min 682 1" "8 f32 sum 4096 1" "8 f32 sum 680 4" "7 f32 sum 680 2" "6 bf16 sum 1000 1" "8 i64 sum 682 2"; do
    set -- $cfg
    POLAR_JITTER_NS=$j timeout 60 python scripts/experiments/repro_ulf.py $1 $2 $3 ring $4 $5 100 2>&1 | grep -E "^(OK|FAIL)" | cut -c1-90 | sed "s/^/jit=$j /"
  done
done
POLAR_STRESS_S=420 POLAR_TIMEOUT_MS=20000 timeout 900 python -m pytest tests/test_gpu_stress.py -x -q -s 2>&1 | tail -4
