#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
for L in cur b8 s8 b8s8 ll4; do
  if [ $L = cur ]; then unset POLAR_LIB; else export POLAR_LIB=build/variants/libpolar_$L.so; fi
  timeout 600 python scripts/sweep.py --n 8 --dtype f32 --sizes 1M,16M,128M --algos ring:simple,tree:simple,ring:ll128,ring:ll,oneshot:simple,twoshot:ll128 --nch 18 --iters 20 > gpurun_out/ring_$L.jsonl 2>&1
  python -c "
import json
r=[json.loads(l) for l in open('gpurun_out/ring_$L.jsonl') if l.startswith('{')]
print('$L', [(x['algo']+':'+x['proto'], x['bytes']>>20, x.get('busbw_gbs')) for x in r])"
done
unset POLAR_LIB
for c in 4194304 8388608 16777216 33554432; do
  POLAR_HOST_CHUNK=$c python -c "
import torch, time, json, synth
from paper_2603_11438_b200 import polar as L
n=8; count=(128<<20)//4
comm=L.Comm.virtual(n,0)
dev=[torch.empty(count, device='cuda') for _ in range(n)]
host=[torch.empty(count).uniform_(-1,1).pin_memory() for _ in range(n)]
comm.allreduce_host(host, dev)
torch.cuda.synchronize(); t0=time.perf_counter()
for _ in range(5): comm.allreduce_host(host, dev)
print(json.dumps({'chunk': $c, 'ms': round((time.perf_counter()-t0)/5*1e3, 2)}))"
done
