#!/bin/bash
# The real-comm random stress (tests/mp_worker_stress.py) with 8 processes sharing
# GPU 0 under MPS (concurrent, like ranks on a node; peers are local HBM).
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
export CUDA_MPS_PIPE_DIRECTORY=/tmp/polar_mps_pipe CUDA_MPS_LOG_DIRECTORY=/tmp/polar_mps_log
mkdir -p $CUDA_MPS_PIPE_DIRECTORY $CUDA_MPS_LOG_DIRECTORY
nvidia-cuda-mps-control -d && echo "mps up"
export POLAR_TIMEOUT_MS=60000 POLAR_STRESS_S=${POLAR_STRESS_S:-150} POLAR_STRESS_POLICY=${POLAR_STRESS_POLICY-policies/mps_cap16.json}
for j in 0 3000; do
  POLAR_JITTER_NS=$j timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 \
    --master-port $((29600 + j % 97)) tests/mp_worker_stress.py gpurun_out/mps_stress_j$j.json > gpurun_out/mps_stress_j$j.log 2>&1
  echo "jitter=$j rc=$?"
  python -c "
import json; r=json.load(open('gpurun_out/mps_stress_j$j.json'))
print({'ranks': len(r), 'calls_per_rank': r[0]['calls'], 'bad': sum(len(x['bad']) for x in r), 'kinds': len(r[0]['kinds']), 'll128_probe': r[0]['ll128_probe']})"
done
echo quit | nvidia-cuda-mps-control
