#!/bin/bash
# compute-sanitizer memcheck over the REAL-comm path: 2 processes (CUDA IPC) under MPS,
# each process under memcheck, running tests/mp_worker.py (every algorithm x protocol,
# registrations, bounce pipeline, graphs, LL128 cross-rank probe, decision latch)
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
export CUDA_MPS_PIPE_DIRECTORY=/tmp/polar_mps_pipe CUDA_MPS_LOG_DIRECTORY=/tmp/polar_mps_log
mkdir -p $CUDA_MPS_PIPE_DIRECTORY $CUDA_MPS_LOG_DIRECTORY
nvidia-cuda-mps-control -d && echo "mps up"
export POLAR_TIMEOUT_MS=600000 POLAR_BOUNCE=1048576 POLAR_NVLS=0
for tool in memcheck synccheck; do
  rm -f gpurun_out/r02q_${tool}_*.log
  timeout 2400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29711 \
    --no-python compute-sanitizer --tool $tool --error-exitcode 9 --log-file gpurun_out/r02q_${tool}_%p.log \
    python tests/mp_worker.py gpurun_out/r02q_mp_$tool.json > gpurun_out/r02q_run_$tool.log 2>&1
  echo "$tool rc=$?"
  grep -h "ERROR SUMMARY" gpurun_out/r02q_${tool}_*.log
  python -c "
import json; r=json.load(open('gpurun_out/r02q_mp_$tool.json')); bad=[x for x in r if not (x['ok'] and x['identical'])]
print(len(r), 'results', len(bad), 'bad')"
done
echo quit | nvidia-cuda-mps-control
