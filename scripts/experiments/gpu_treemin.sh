#!/bin/bash
# tree Simple: plain kernel below 16 KiB per channel (cur) vs always warp-specialised (nomin)
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
export POLAR_TIMEOUT_MS=5000
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multiproc.py tests/test_gpu_faults.py tests/test_gpu_graphs.py -q -x --timeout=300 -k "tree or back_to_back or multiprocess or unit_sizes or jitter or graph" > gpurun_out/treemin_parity.log 2>&1
echo "parity: $(tail -n 1 gpurun_out/treemin_parity.log)"
for i in 1 2; do
  for L in cur nomin; do
    if [ $L = cur ]; then unset POLAR_LIB; else export POLAR_LIB=build/variants/libpolar_$L.so; fi
    timeout 600 python scripts/sweep.py --n 8 --dtype f32 --sizes 4K,64K,256K,1M,8M --algos tree:simple --nch 4,18 --iters 20 --graph > gpurun_out/treemin_${L}_$i.jsonl 2>&1
    python -c "
import json
r=[json.loads(l) for l in open('gpurun_out/treemin_${L}_$i.jsonl') if l.startswith('{')]
print('$L', $i, [(x['nch'], x['bytes']>>10, x.get('us')) for x in r])"
  done
done
