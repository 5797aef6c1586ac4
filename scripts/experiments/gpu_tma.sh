#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
for n in 2 4 8; do for t in 0 1; do
  POLAR_TWOSHOT_TMA=$t timeout 600 python scripts/sweep.py --n $n --dtype bf16 --sizes 16M,64M,256M,1G --algos twoshot:simple --nch 32 --iters 10 > gpurun_out/tma_${n}_$t.jsonl 2>&1
  python -c "
import json
r=[json.loads(l) for l in open('gpurun_out/tma_${n}_$t.jsonl') if l.startswith('{')]
print('n=$n tma=$t', [(x['bytes']>>20, x.get('busbw_gbs')) for x in r])"
done; done
