#!/bin/bash
# ncu --set full of the ring Simple kernels at 8 x 128 MiB f32: warp-specialised LDG vs TMA-staged
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
export POLAR_TIMEOUT_MS=20000 AB_SIZES_MIB=128 AB_DTYPES=f32
for v in "POLAR_RING_TMA=0" "POLAR_RING_TMA=1;POLAR_RING_TMA_FLAGS=1"; do
  tag=$(echo $v | tr ';=' '__')
  AB_VARIANTS="$v" timeout 900 ncu --set full --clock-control none --import-source on -k regex:allreduce_kernel -s 2 -c 1 \
    -f -o gpurun_out/prof_ring_$tag python scripts/experiments/exp_ring_tma.py > gpurun_out/ncu_ring_$tag.log 2>&1
  echo "$v rc=$?"
done
