#!/bin/bash
# A/B: discard.global.L2 of consumed Simple FIFO / staging lines (ring, tree,
# one-shot Simple; 8 virtual ranks, f32) vs the POLAR_DISCARD=0 build; parity subset first
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
export POLAR_TIMEOUT_MS=5000
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_graphs.py -q -x -k "simple or graph or back_to_back or policy" > gpurun_out/discard_parity.log 2>&1
tail -2 gpurun_out/discard_parity.log
for i in 1 2; do
  for L in cur nodiscard; do
    if [ $L = cur ]; then unset POLAR_LIB; else export POLAR_LIB=build/variants/libpolar_$L.so; fi
    timeout 600 python scripts/sweep.py --n 8 --dtype f32 --sizes 1M,8M,32M,128M --algos ring:simple,tree:simple,oneshot:simple --nch 18 --iters 10 --graph > gpurun_out/discard_${L}_$i.jsonl 2>&1
    python -c "
import json
r=[json.loads(l) for l in open('gpurun_out/discard_${L}_$i.jsonl') if l.startswith('{')]
print('$L', $i, [(x['algo'], x['bytes']>>20, x.get('us'), x.get('busbw_gbs')) for x in r])"
  done
done
unset POLAR_LIB
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:allreduce_kernel -c 6 --csv \
  python scripts/sweep.py --n 8 --dtype f32 --sizes 128M --algos ring:simple,tree:simple,oneshot:simple --nch 18 --iters 1 --warm 1 > gpurun_out/discard_ncu.csv 2>&1
grep -E "dram__bytes|gpu__time" gpurun_out/discard_ncu.csv | cut -c1-400 | tail -18
