#!/bin/bash
# ncu --set full of the warp-specialised ring Simple (f32, 8 virtual ranks, 128 MiB)
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:allreduce_kernel -s 2 -c 1 -f -o gpurun_out/prof_ring_ws \
  python scripts/sweep.py --n 8 --dtype f32 --sizes 128M --algos ring:simple --nch 18 --iters 1 --warm 1 > gpurun_out/ncu_ring_ws.log 2>&1
echo "ncu rc=$?"
