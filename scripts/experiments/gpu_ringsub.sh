#!/bin/bash
# ring Simple sub-slice flags (POLAR_RING_SUB = 1 / 2 / 4 sub-slices per FIFO slot):
# parity of every ring case under each build, then busBW (8 virtual ranks, f32, CUDA graph)
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
export POLAR_TIMEOUT_MS=5000
for L in cur rsub2 rsub4; do
  if [ $L = cur ]; then unset POLAR_LIB; else export POLAR_LIB=build/variants/libpolar_$L.so; fi
  timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "ring or back_to_back" > gpurun_out/ringsub_parity_$L.log 2>&1
  echo "$L parity: $(tail -1 gpurun_out/ringsub_parity_$L.log)"
done
for i in 1 2; do
  for L in cur rsub2 rsub4; do
    if [ $L = cur ]; then unset POLAR_LIB; else export POLAR_LIB=build/variants/libpolar_$L.so; fi
    for sl in 131072 262144; do
      POLAR_RING_SLOT=$sl timeout 600 python scripts/sweep.py --n 8 --dtype f32 --sizes 1M,8M,32M,128M --algos ring:simple --nch 18 --iters 10 --graph > gpurun_out/ringsub_${L}_${sl}_$i.jsonl 2>&1
      python -c "
import json
r=[json.loads(l) for l in open('gpurun_out/ringsub_${L}_${sl}_$i.jsonl') if l.startswith('{')]
print('$L', $sl, $i, [(x['bytes']>>20, x.get('us'), x.get('busbw_gbs')) for x in r])"
    done
  done
done
