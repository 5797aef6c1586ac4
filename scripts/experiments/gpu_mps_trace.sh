#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
export CUDA_MPS_PIPE_DIRECTORY=/tmp/polar_mps_pipe CUDA_MPS_LOG_DIRECTORY=/tmp/polar_mps_log
mkdir -p $CUDA_MPS_PIPE_DIRECTORY $CUDA_MPS_LOG_DIRECTORY
nvidia-cuda-mps-control -d && echo "mps up"
export POLAR_TIMEOUT_MS=20000
for cfg in "8 16 128" "8 18 128" "8 16 4" "4 16 128"; do set -- $cfg
  NCH=$2 MIB=$3 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $1 --master-addr 127.0.0.1 \
    --master-port $((29700 + $1 + $2)) scripts/experiments/mps_trace.py 2>/dev/null | grep '^{'
done
echo quit | nvidia-cuda-mps-control
