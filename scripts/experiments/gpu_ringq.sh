#!/bin/bash
# ring WS: sub-slices per slot RQ = 2 (cur) / 3 / 4 at slot sizes giving whole batches per unit
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
export POLAR_TIMEOUT_MS=5000
for L in wsq3 wsq4; do
  POLAR_LIB=build/variants/libpolar_$L.so POLAR_RING_SLOT=245760 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "ring" > gpurun_out/ringq_parity_$L.log 2>&1
  echo "$L parity: $(tail -1 gpurun_out/ringq_parity_$L.log)"
done
for i in 1 2; do
  for cfg in "cur 122880" "wsq3 184320" "wsq3 368640" "wsq4 122880" "wsq4 245760"; do
    set -- $cfg; L=$1; sl=$2
    if [ $L = cur ]; then unset POLAR_LIB; else export POLAR_LIB=build/variants/libpolar_$L.so; fi
    POLAR_RING_SLOT=$sl timeout 600 python scripts/sweep.py --n 8 --dtype f32 --sizes 1M,8M,32M,128M --algos ring:simple --nch 18 --iters 10 --graph > gpurun_out/ringq_${L}_${sl}_$i.jsonl 2>&1
    POLAR_RING_SLOT=$sl timeout 600 python scripts/sweep.py --n 8 --dtype bf16 --sizes 128M --algos ring:simple --nch 18 --iters 10 --graph >> gpurun_out/ringq_${L}_${sl}_$i.jsonl 2>&1
    python -c "
import json
r=[json.loads(l) for l in open('gpurun_out/ringq_${L}_${sl}_$i.jsonl') if l.startswith('{')]
print('$L', $sl, $i, [(x['dtype'], x['bytes']>>20, x.get('us')) for x in r])"
  done
done
