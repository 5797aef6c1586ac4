#!/bin/bash
# ring / tree FIFO slot size sweep (runtime env, virtual ranks)
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
for sl in 32768 65536 131072 262144 524288; do
  POLAR_RING_SLOT=$sl POLAR_TREE_SLOT=$sl POLAR_RING128_SLOT=$sl timeout 600 python scripts/sweep.py --n 8 --dtype f32 --sizes 1M,16M,128M --algos ring:simple,tree:simple,ring:ll128 --nch 32 --iters 10 > gpurun_out/rs_$sl.jsonl 2>&1
  python -c "
import json
r=[json.loads(l) for l in open('gpurun_out/rs_$sl.jsonl') if l.startswith('{')]
print($sl, [(x['algo']+':'+x['proto'], x['bytes']>>20, x.get('busbw_gbs')) for x in r])"
done
