#!/bin/bash
# direct ReduceScatter / AllGather / Broadcast: dynamic chunks (cur) vs static slices (dirstatic)
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
export POLAR_TIMEOUT_MS=5000
timeout 900 python -m pytest tests/test_gpu_collectives.py tests/test_gpu_multiproc.py tests/test_gpu_graphs.py -q -x --timeout=300 > gpurun_out/dyn_parity.log 2>&1
echo "parity: $(tail -n 1 gpurun_out/dyn_parity.log)"
for i in 1 2; do
  for L in cur dirstatic; do
    if [ $L = cur ]; then unset POLAR_LIB; else export POLAR_LIB=build/variants/libpolar_$L.so; fi
    timeout 900 python scripts/report_configs.py --configs f4 > gpurun_out/dyn_${L}_$i.jsonl 2>/dev/null
    python -c "
import json
r=[json.loads(l) for l in open('gpurun_out/dyn_${L}_$i.jsonl') if l.startswith('{') and 'F4' in l]
print('$L', $i, [(x['bytes']>>20, x['reduce_scatter']['busbw_gbs'], x['all_gather']['busbw_gbs'], x['broadcast']['busbw_gbs']) for x in r])"
  done
done
