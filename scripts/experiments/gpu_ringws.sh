#!/bin/bash
# warp-specialised ring Simple (POLAR_RING_WS): parity + faults + multiprocess,
# then A/B vs the plain ring (ringold) and 1 / 4 sub-slices (wsq1 / wsq4)
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
export POLAR_TIMEOUT_MS=5000
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_faults.py tests/test_gpu_graphs.py tests/test_gpu_multiproc.py -q -x --timeout=300 -k "ring or back_to_back or fault or timeout or graph or multiprocess or policy" > gpurun_out/ringws_parity.log 2>&1
echo "parity: $(tail -1 gpurun_out/ringws_parity.log)"
grep -E "FAIL|Error" gpurun_out/ringws_parity.log | head -5
for i in 1 2; do
  for L in cur ringold wsq1 wsq4; do
    if [ $L = cur ]; then unset POLAR_LIB; else export POLAR_LIB=build/variants/libpolar_$L.so; fi
    timeout 600 python scripts/sweep.py --n 8 --dtype f32 --sizes 1M,8M,32M,128M --algos ring:simple --nch 18 --iters 10 --graph > gpurun_out/ringws_${L}_$i.jsonl 2>&1
    timeout 600 python scripts/sweep.py --n 8 --dtype bf16 --sizes 128M --algos ring:simple --nch 18 --iters 10 --graph >> gpurun_out/ringws_${L}_$i.jsonl 2>&1
    python -c "
import json
r=[json.loads(l) for l in open('gpurun_out/ringws_${L}_$i.jsonl') if l.startswith('{')]
print('$L', $i, [(x['dtype'], x['bytes']>>20, x.get('us'), x.get('busbw_gbs')) for x in r])"
  done
done
