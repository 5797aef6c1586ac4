#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
export CUDA_MPS_PIPE_DIRECTORY=/tmp/polar_mps_pipe CUDA_MPS_LOG_DIRECTORY=/tmp/polar_mps_log
mkdir -p $CUDA_MPS_PIPE_DIRECTORY $CUDA_MPS_LOG_DIRECTORY
nvidia-cuda-mps-control -d && echo "mps up"
export POLAR_BENCH_SHARE_GPU=1 POLAR_TIMEOUT_MS=10000
for cfg in "PDL0:POLAR_PDL=0" "PDL1:POLAR_PDL=1"; do
  name=${cfg%%:*}; envs=${cfg#*:}
  env $envs timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
    --master-port 29611 bench.py --gpus 4 --steps 10 --warmup 3 --policy policies/mps_cap16.json \
    > gpurun_out/mpsdbg_$name.json 2> gpurun_out/mpsdbg_$name.err
  echo "$name rc=$?"; grep -o "POLAR_E[A-Z]*" gpurun_out/mpsdbg_$name.err | sort | uniq -c
  python -c "import json; d=json.load(open('gpurun_out/mpsdbg_$name.json')); print(d['value'])" 2>/dev/null
done
cat $CUDA_MPS_LOG_DIRECTORY/*.log 2>/dev/null | tail -15
echo quit | nvidia-cuda-mps-control
