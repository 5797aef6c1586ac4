#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
export POLAR_TIMEOUT_MS=20000
timeout 1200 python -m pytest tests/test_gpu_multiproc.py tests/test_gpu_bench.py tests/test_gpu_nvls.py -q -x -rs > gpurun_out/r02g_tests.log 2>&1; echo "tests rc=$?"; tail -4 gpurun_out/r02g_tests.log
for N in 2 3; do
  POLAR_BENCH_SHARE_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $((29500+N)) bench.py --gpus $N --steps 20 --warmup 3 > gpurun_out/r02g_bench_shared$N.json 2> gpurun_out/r02g_bench_shared$N.err; echo "bench N=$N rc=$?"
  python -c "
import json; d=json.loads([l for l in open('gpurun_out/r02g_bench_shared$N.json') if l.startswith('{')][0])
print('value', d['value'], 'parity', d['parity']['ok'], 'unreg', d.get('unregistered'), 'll128', d.get('ll128_probe'))"
done
