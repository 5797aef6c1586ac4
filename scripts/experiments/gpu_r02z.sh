#!/bin/bash
# ncu --set full of the cluster ring at 128 MiB (f32 and bf16)
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
for dt in f32 bf16; do
  CL_DT=$dt CL_MIB=128 timeout 600 ncu --set full --clock-control none --import-source on -k regex:${CL_KERNEL:-ring_cluster} -s 1 -c 1 -f -o gpurun_out/prof_cl_$dt python scripts/experiments/exp_cl_once.py > gpurun_out/r02z_ncu_$dt.log 2>&1; echo "ncu $dt rc=$?"
done
