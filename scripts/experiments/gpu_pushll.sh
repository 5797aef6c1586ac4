#!/bin/bash
# LL push loops (one-shot / two-shot LL): 2 (cur) / 4 / 8 packs per thread per iteration
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
export POLAR_TIMEOUT_MS=5000
for L in push4 push8; do
  POLAR_LIB=build/variants/libpolar_$L.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "oneshot or twoshot" > gpurun_out/pushll_parity_$L.log 2>&1
  echo "$L parity: $(tail -n 1 gpurun_out/pushll_parity_$L.log)"
done
for i in 1 2; do
  for L in cur push4 push8; do
    if [ $L = cur ]; then unset POLAR_LIB; else export POLAR_LIB=build/variants/libpolar_$L.so; fi
    timeout 600 python scripts/sweep.py --n 8 --dtype f32 --sizes 1K,16K,64K,256K,1M --algos oneshot:ll,twoshot:ll --nch 4,18 --iters 20 --graph > gpurun_out/pushll_${L}_$i.jsonl 2>&1
    python -c "
import json
r=[json.loads(l) for l in open('gpurun_out/pushll_${L}_$i.jsonl') if l.startswith('{')]
print('$L', $i, [(x['algo'], x['nch'], x['bytes']>>10, x.get('us')) for x in r])"
  done
done
