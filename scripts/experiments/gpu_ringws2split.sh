#!/bin/bash
# ring Simple with split sync warps (poller + publisher; POLAR_RING_WS=2), RQ = 2 / 1, vs the adopted ring WS
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
export POLAR_TIMEOUT_MS=5000
for L in ws2q2 ws2q1; do
  POLAR_LIB=build/variants/libpolar_$L.so POLAR_RING_SLOT=114688 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multiproc.py tests/test_gpu_faults.py -q -x --timeout=300 -k "ring or back_to_back or multiprocess or unit_sizes or fault or timeout" > gpurun_out/split_parity_$L.log 2>&1
  echo "$L parity: $(tail -n 1 gpurun_out/split_parity_$L.log)"
done
for i in 1 2; do
  for cfg in "cur 122880" "ws2q2 114688" "ws2q2 229376" "ws2q1 114688" "ws2q1 229376"; do
    set -- $cfg; L=$1; sl=$2
    if [ $L = cur ]; then unset POLAR_LIB; else export POLAR_LIB=build/variants/libpolar_$L.so; fi
    POLAR_RING_SLOT=$sl timeout 600 python scripts/sweep.py --n 8 --dtype f32 --sizes 1M,8M,32M,128M --algos ring:simple --nch 18 --iters 10 --graph > gpurun_out/split_${L}_${sl}_$i.jsonl 2>&1
    POLAR_RING_SLOT=$sl timeout 600 python scripts/sweep.py --n 8 --dtype bf16 --sizes 128M --algos ring:simple --nch 18 --iters 10 --graph >> gpurun_out/split_${L}_${sl}_$i.jsonl 2>&1
    python -c "
import json
r=[json.loads(l) for l in open('gpurun_out/split_${L}_${sl}_$i.jsonl') if l.startswith('{')]
print('$L', $sl, $i, [(x['dtype'], x['bytes']>>20, x.get('us')) for x in r])"
  done
done
