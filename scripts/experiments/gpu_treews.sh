#!/bin/bash
# warp-specialised tree Simple (POLAR_TREE_WS): parity + faults + multiprocess,
# then A/B vs the plain tree (treeold, 128 KiB slots)
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
export POLAR_TIMEOUT_MS=5000
POLAR_LIB=build/variants/libpolar_treeq1.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_faults.py tests/test_gpu_graphs.py tests/test_gpu_multiproc.py -q -x --timeout=300 -k "tree or back_to_back or fault or timeout or graph or multiprocess or policy" > gpurun_out/treews_parity.log 2>&1
echo "parity: $(tail -1 gpurun_out/treews_parity.log)"
grep -E "FAIL|Error" gpurun_out/treews_parity.log | head -5
for i in 1 2; do
  for cfg in "cur 122880" "treeq1 122880" "treeold 131072"; do
    set -- $cfg; L=$1; sl=$2
    if [ $L = cur ]; then unset POLAR_LIB; else export POLAR_LIB=build/variants/libpolar_$L.so; fi
    POLAR_TREE_SLOT=$sl timeout 600 python scripts/sweep.py --n 8 --dtype f32 --sizes 4K,1M,8M,32M,128M --algos tree:simple --nch 18 --iters 10 --graph > gpurun_out/treews_${L}_$i.jsonl 2>&1
    POLAR_TREE_SLOT=$sl timeout 600 python scripts/sweep.py --n 8 --dtype bf16 --sizes 128M --algos tree:simple --nch 18 --iters 10 --graph >> gpurun_out/treews_${L}_$i.jsonl 2>&1
    python -c "
import json
r=[json.loads(l) for l in open('gpurun_out/treews_${L}_$i.jsonl') if l.startswith('{')]
print('$L', $i, [(x['dtype'], x['bytes']>>10, x.get('us'), x.get('busbw_gbs')) for x in r])"
  done
done
