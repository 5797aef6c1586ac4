#!/bin/bash
# The REAL-comm path (one process per rank, CUDA-IPC peer mappings, sys-scope
# flags, entry/exit handshakes, per-process launches) benchmarked on ONE GPU:
# N processes share GPU 0 concurrently under MPS (without MPS, contexts
# time-slice and cross-process spin-waits crawl).  Peers are local HBM, not
# NVLink.  Channels capped at 16 so N x nch CTAs stay co-resident (N <= 8).
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
export CUDA_MPS_PIPE_DIRECTORY=/tmp/polar_mps_pipe CUDA_MPS_LOG_DIRECTORY=/tmp/polar_mps_log
mkdir -p $CUDA_MPS_PIPE_DIRECTORY $CUDA_MPS_LOG_DIRECTORY
nvidia-cuda-mps-control -d && echo "mps up"
export POLAR_BENCH_SHARE_GPU=1 POLAR_TIMEOUT_MS=20000
for n in ${@:-2 4 8}; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port $((29500 + n)) bench.py --gpus $n --steps 50 --warmup 5 --policy policies/mps_cap16.json \
    > gpurun_out/mps_bench_$n${TAG:-}.json 2> gpurun_out/mps_bench_$n${TAG:-}.err
  echo "n=$n rc=$?"
  python -c "
import json
d=json.loads([l for l in open('gpurun_out/mps_bench_$n${TAG:-}.json') if l.startswith('{')][0])
print({k: d[k] for k in ('value','ms_per_step','n_gpus')}, d['decision'], d['roofline']['hbm']['frac'], d['p2p_probe'], d.get('unregistered'), d['parity']['ok'])" 2>&1 | tail -2
done
echo quit | nvidia-cuda-mps-control
