#!/bin/bash
# round 2: cluster ring ablations (profile build): no DSMEM stores / no HBM stores / 16 compute warps
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
for L in clprof abl1 abl2 w16; do
  echo "== $L"; POLAR_LIB=build/variants/libpolar_$L.so timeout 120 python scripts/experiments/exp_cl_prof.py 2>&1 | tail -2
done | tee gpurun_out/r02v_abl.txt
