#!/bin/bash
# tree WS with the runtime unit size (half slots at <= 4 slots per channel, else whole)
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
export POLAR_TIMEOUT_MS=5000
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_faults.py tests/test_gpu_graphs.py tests/test_gpu_multiproc.py -q -x --timeout=300 -k "tree or ring or back_to_back or fault or timeout or graph or multiprocess or policy or unit_sizes" > gpurun_out/treews2_parity.log 2>&1
echo "parity: $(tail -1 gpurun_out/treews2_parity.log)"
grep -E "FAIL|Error" gpurun_out/treews2_parity.log | head -5
for i in 1 2; do
  for cfg in "cur 122880"; do
    set -- $cfg; L=$1; sl=$2
    if [ $L = cur ]; then unset POLAR_LIB; else export POLAR_LIB=build/variants/libpolar_$L.so; fi
    POLAR_TREE_SLOT=$sl timeout 600 python scripts/sweep.py --n 8 --dtype f32 --sizes 4K,64K,1M,4M,8M,32M,128M --algos tree:simple --nch 18 --iters 10 --graph > gpurun_out/treews2_${L}_$i.jsonl 2>&1
    POLAR_TREE_SLOT=$sl timeout 600 python scripts/sweep.py --n 8 --dtype bf16 --sizes 128M --algos tree:simple --nch 18 --iters 10 --graph >> gpurun_out/treews2_${L}_$i.jsonl 2>&1
    python -c "
import json
r=[json.loads(l) for l in open('gpurun_out/treews2_${L}_$i.jsonl') if l.startswith('{')]
print('$L', $i, [(x['dtype'], x['bytes']>>10, x.get('us')) for x in r])"
  done
done
