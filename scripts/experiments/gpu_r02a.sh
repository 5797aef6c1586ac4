#!/bin/bash
# round 2 first contact: fabric/multicast diagnosis + GPU tests at HEAD
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
O=gpurun_out/r02a_fabric.txt
{
  echo "== nvidia-smi -L"; nvidia-smi -L
  echo "== topo"; nvidia-smi topo -m
  echo "== nvlink status"; nvidia-smi nvlink -s 2>&1 | head -40
  echo "== fabric (nvidia-smi -q)"; nvidia-smi -q | grep -i -A6 "fabric"
  echo "== /dev"; ls -la /dev | grep -i nvidia
  echo "== imex"; ls /dev/nvidia-caps-imex-channels 2>&1; cat /proc/driver/nvidia/capabilities/fabric-imex-mgmt 2>&1 | head
  echo "== fm processes"; ps aux | grep -i -E "fabric|imex" | grep -v grep
  echo "== CUDA_VISIBLE_DEVICES=$CUDA_VISIBLE_DEVICES"
  echo "== cpu"; grep -m1 "model name" /proc/cpuinfo; nproc
  echo "== nccl libs"; python -c "import nvidia.nccl, os; d=os.path.dirname(nvidia.nccl.__file__); print(d); print(os.listdir(os.path.join(d,'lib')))" 2>&1
} > $O 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/probe_mc scripts/probe_multicast.cu -lcuda >> $O 2>&1
timeout 120 /tmp/probe_mc > gpurun_out/r02a_probe_multicast.txt 2>&1; echo "probe rc=$?" >> gpurun_out/r02a_probe_multicast.txt
cat gpurun_out/r02a_probe_multicast.txt | tail -30
timeout 1800 python -m pytest tests -m gpu -q -x --timeout=600 > gpurun_out/r02a_pytest_gpu.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/r02a_pytest_gpu.log
