#!/bin/bash
# ring / tree WS: L2 bulk prefetch of the next own range by the sync warp (cur) vs none (nopf)
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
export POLAR_TIMEOUT_MS=5000
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multiproc.py tests/test_gpu_graphs.py -q -x --timeout=300 -k "tree or ring or back_to_back or graph or multiprocess or unit_sizes or edges" > gpurun_out/wspf_parity.log 2>&1
echo "parity: $(tail -1 gpurun_out/wspf_parity.log)"
for i in 1 2; do
  for L in cur nopf; do
    if [ $L = cur ]; then unset POLAR_LIB; else export POLAR_LIB=build/variants/libpolar_$L.so; fi
    timeout 600 python scripts/sweep.py --n 8 --dtype f32 --sizes 1M,8M,32M,128M --algos ring:simple,tree:simple --nch 18 --iters 10 --graph > gpurun_out/wspf_${L}_$i.jsonl 2>&1
    timeout 600 python scripts/sweep.py --n 8 --dtype bf16 --sizes 128M --algos ring:simple,tree:simple --nch 18 --iters 10 --graph >> gpurun_out/wspf_${L}_$i.jsonl 2>&1
    python -c "
import json
r=[json.loads(l) for l in open('gpurun_out/wspf_${L}_$i.jsonl') if l.startswith('{')]
print('$L', $i, [(x['algo'], x['dtype'], x['bytes']>>20, x.get('us')) for x in r])"
  done
done
