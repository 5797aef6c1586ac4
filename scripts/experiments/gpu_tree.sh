#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
export POLAR_TIMEOUT_MS=5000
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_faults.py -q -x -k "tree or ring or jitter" --timeout=600 2>&1 | tail -3
for L in cur old; do
  if [ $L = cur ]; then unset POLAR_LIB; else export POLAR_LIB=build/variants/libpolar_$L.so; fi
  timeout 600 python scripts/sweep.py --n 8 --dtype f32 --sizes 1K,64K,1M,16M,128M --algos tree:ll,tree:simple,ring:ll,ring:ll128,ring:simple --nch 16 --graph --iters 20 > gpurun_out/tree_$L.jsonl 2>&1
  python -c "
import json
r=[json.loads(l) for l in open('gpurun_out/tree_$L.jsonl') if l.startswith('{')]
print('$L', [(x['proto'], x['bytes'], x.get('us')) for x in r])"
done
