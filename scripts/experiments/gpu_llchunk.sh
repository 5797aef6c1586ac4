#!/bin/bash
# LL / LL128 staging chunk sweep (runtime env, 8 virtual ranks, f32): two-shot
# (POLAR_TSLL_CHUNK) and one-shot (POLAR_OSLL_CHUNK) at 128 KiB - 32 MiB
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
for ch in 65536 262144 1048576; do
  POLAR_TSLL_CHUNK=$ch POLAR_OSLL_CHUNK=$((ch*4)) timeout 600 python scripts/sweep.py --n 8 --dtype f32 \
    --sizes 128K,512K,2M,8M,32M --algos twoshot:ll,twoshot:ll128,oneshot:ll,oneshot:ll128 --nch 8,18 --iters 10 --graph \
    > gpurun_out/llchunk_$ch.jsonl 2>&1
  python -c "
import json
r=[json.loads(l) for l in open('gpurun_out/llchunk_$ch.jsonl') if l.startswith('{')]
best={}
for x in r:
  k=(x['algo']+':'+x['proto'], x['bytes']>>10)
  if 'us' in x and (k not in best or x['us']<best[k]): best[k]=x['us']
print($ch, sorted(best.items()))"
done
