#!/bin/bash
# A/B: bench with the current lib vs a variant lib (build/variants/libpolar_$1.so), interleaved
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
V=${1:-old}
for i in 1 2; do
  for L in cur $V; do
    if [ $L = cur ]; then unset POLAR_LIB; else export POLAR_LIB=build/variants/libpolar_$L.so; fi
    timeout 600 python bench.py --steps 200 > gpurun_out/ab_${L}_$i.json 2>/dev/null
    python -c "
import json; d=json.load(open('gpurun_out/ab_${L}_$i.json'))
print('$L', $i, d['value'], d['ms_per_step'], {k: v['us'] for k, v in d['c2_sweep'].items()})"
  done
done
