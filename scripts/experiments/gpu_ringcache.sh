#!/bin/bash
# ring WS: fill and credit polled by two lanes in parallel, with (cur) / without (nocache) the per-lane cache
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
export POLAR_TIMEOUT_MS=5000
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multiproc.py tests/test_gpu_faults.py -q -x --timeout=300 -k "ring or back_to_back or multiprocess or unit_sizes or fault or timeout" > gpurun_out/ringcache_parity.log 2>&1
echo "parity: $(tail -n 1 gpurun_out/ringcache_parity.log)"
for i in 1 2; do
  for L in cur nocache; do
    if [ $L = cur ]; then unset POLAR_LIB; else export POLAR_LIB=build/variants/libpolar_$L.so; fi
    timeout 600 python scripts/sweep.py --n 8 --dtype f32 --sizes 1M,8M,32M,128M --algos ring:simple --nch 18 --iters 10 --graph > gpurun_out/ringcache_${L}_$i.jsonl 2>&1
    timeout 600 python scripts/sweep.py --n 8 --dtype bf16 --sizes 128M --algos ring:simple --nch 18 --iters 10 --graph >> gpurun_out/ringcache_${L}_$i.jsonl 2>&1
    python -c "
import json
r=[json.loads(l) for l in open('gpurun_out/ringcache_${L}_$i.jsonl') if l.startswith('{')]
print('$L', $i, [(x['dtype'], x['bytes']>>20, x.get('us')) for x in r])"
  done
done
