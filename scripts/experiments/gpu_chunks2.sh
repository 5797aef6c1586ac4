#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
for rep in 1 2; do
for L in cur b512 b768 b1k b1536; do
  if [ $L = cur ]; then unset POLAR_LIB; else export POLAR_LIB=build/variants/libpolar_$L.so; fi
  timeout 600 python scripts/sweep.py --n 8 --dtype f32 --sizes 4M,8M,16M,32M,64M,128M --algos twoshot:simple --nch 32 --iters 50 > gpurun_out/ch2_$L.jsonl 2>&1
  python -c "
import json
r=[json.loads(l) for l in open('gpurun_out/ch2_$L.jsonl') if l.startswith('{')]
print('$L', [(x['bytes']>>20, x['us']) for x in r])"
done
done
