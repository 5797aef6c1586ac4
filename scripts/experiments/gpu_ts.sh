#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
python scripts/experiments/probe_mc2.py > gpurun_out/probe_mc2.txt 2>&1
for L in cur big4k small512 small1k; do
  if [ $L = cur ]; then unset POLAR_LIB; else export POLAR_LIB=build/variants/libpolar_$L.so; fi
  timeout 600 python scripts/sweep.py --n 8 --dtype f32 --sizes 1M,2M,4M,8M,16M,32M,64M,128M --algos twoshot:simple --nch 32 --iters 50 > gpurun_out/ts_$L.jsonl 2>&1
  python -c "
import json
r=[json.loads(l) for l in open('gpurun_out/ts_$L.jsonl') if l.startswith('{')]
print('$L', [(x['bytes']>>20, x['us']) for x in r])"
done
unset POLAR_LIB
for m in 4 16 128; do timeout 300 python scripts/trace_kernel.py --n 8 --mib $m --nch 32 --reps 2; done > gpurun_out/trace_ts.jsonl 2>&1
cat gpurun_out/trace_ts.jsonl
