#!/bin/bash
# ring WS (RQ = 2) vs plain ring at FIFO slot sizes that give whole batch
# iterations per unit (WS: 480 data threads x 4 packs = 1920 packs; plain: 2048)
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
export POLAR_TIMEOUT_MS=5000
for i in 1 2; do
  for cfg in "cur 122880" "cur 245760" "cur 491520" "ringold 131072" "ringold 262144"; do
    set -- $cfg; L=$1; sl=$2
    if [ $L = cur ]; then unset POLAR_LIB; else export POLAR_LIB=build/variants/libpolar_$L.so; fi
    POLAR_RING_SLOT=$sl timeout 600 python scripts/sweep.py --n 8 --dtype f32 --sizes 1M,8M,32M,128M --algos ring:simple --nch 18 --iters 10 --graph > gpurun_out/ringws2_${L}_${sl}_$i.jsonl 2>&1
    POLAR_RING_SLOT=$sl timeout 600 python scripts/sweep.py --n 8 --dtype bf16 --sizes 128M --algos ring:simple --nch 18 --iters 10 --graph >> gpurun_out/ringws2_${L}_${sl}_$i.jsonl 2>&1
    python -c "
import json
r=[json.loads(l) for l in open('gpurun_out/ringws2_${L}_${sl}_$i.jsonl') if l.startswith('{')]
print('$L', $sl, $i, [(x['dtype'], x['bytes']>>20, x.get('us'), x.get('busbw_gbs')) for x in r])"
  done
done
