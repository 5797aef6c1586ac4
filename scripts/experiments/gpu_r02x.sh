#!/bin/bash
# ncu --set full of the cluster ring (second call, 32 MiB f32)
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ring_cluster -s 1 -c 1 -f -o gpurun_out/prof_cl python scripts/experiments/exp_cl_once.py > gpurun_out/r02x_ncu.log 2>&1; echo "ncu rc=$?"
tail -3 gpurun_out/r02x_ncu.log
