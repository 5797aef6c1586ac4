#!/bin/bash
# real-comm path at the north_star rank count: 8 processes on one GPU under MPS
# (concurrent contexts), full multi-process parity suites + the N=8 bench line
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
export CUDA_MPS_PIPE_DIRECTORY=/tmp/polar_mps_pipe CUDA_MPS_LOG_DIRECTORY=/tmp/polar_mps_log
mkdir -p $CUDA_MPS_PIPE_DIRECTORY $CUDA_MPS_LOG_DIRECTORY
nvidia-cuda-mps-control -d && echo "mps up"
export POLAR_TIMEOUT_MS=60000 POLAR_POLICY=$PWD/policies/mps_cap16.json
for w in ${WORKERS:-mp_worker mp_worker_c2}; do
  timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 --master-port 29611 \
    tests/$w.py gpurun_out/r02k_${w}_n8.json > gpurun_out/r02k_${w}_n8.log 2>&1
  echo "$w n=8 rc=$?"
  python -c "
import json; r=json.load(open('gpurun_out/r02k_${w}_n8.json'))
bad=[x for x in r if not (x['ok'] and x['identical'])]
print(len(r), 'results,', len(bad), 'bad', bad[:3])" 2>&1 | tail -2
done
unset POLAR_POLICY
[ -n "$NOBENCH" ] || TAG=_r02k bash scripts/gpu_mps_bench.sh 8
echo quit | nvidia-cuda-mps-control
