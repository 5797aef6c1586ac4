#!/bin/bash
# round 2: cluster transport tests + the full GPU suite + bench
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
export POLAR_TIMEOUT_MS=10000
timeout 900 python -m pytest tests/test_gpu_cluster.py -x -q > gpurun_out/r02bb_cluster.log 2>&1; tail -5 gpurun_out/r02bb_cluster.log
timeout 1500 python -m pytest tests -m gpu -q ${PYARGS:-} > gpurun_out/r02bb_gpu.log 2>&1; tail -5 gpurun_out/r02bb_gpu.log
timeout 600 python bench.py > gpurun_out/r02bb_bench.json 2> gpurun_out/r02bb_bench.err; echo "bench rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/r02bb_bench.json'))
print(d['value'], d['roofline']['frac'], d['parity']['ok'])
for k,v in d.get('algorithms',{}).items(): print(k, v)
"
