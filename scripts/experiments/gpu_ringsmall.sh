#!/bin/bash
# ring Simple at small sizes: warp-specialised (cur) vs plain (ringplain, 128 KiB slots)
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
export POLAR_TIMEOUT_MS=5000
for i in 1 2; do
  for cfg in "cur 122880" "ringplain 131072"; do
    set -- $cfg; L=$1; sl=$2
    if [ $L = cur ]; then unset POLAR_LIB; else export POLAR_LIB=build/variants/libpolar_$L.so; fi
    POLAR_RING_SLOT=$sl timeout 600 python scripts/sweep.py --n 8 --dtype f32 --sizes 4K,64K,256K,1M,4M --algos ring:simple --nch 4,18 --iters 20 --graph > gpurun_out/ringsmall_${L}_$i.jsonl 2>&1
    python -c "
import json
r=[json.loads(l) for l in open('gpurun_out/ringsmall_${L}_$i.jsonl') if l.startswith('{')]
print('$L', $i, [(x['nch'], x['bytes']>>10, x.get('us')) for x in r])"
  done
done
