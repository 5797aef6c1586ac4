#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
export POLAR_TIMEOUT_MS=5000
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "matrix_sum or edges or back_to_back or default or policy" --timeout=600 2>&1 | tail -2
bash scripts/gpu_ab.sh block
for m in 4 128; do timeout 300 python scripts/trace_kernel.py --n 8 --mib $m --nch 32 --reps 1; done 2>&1
timeout 600 python scripts/sweep.py --n 8 --dtype f32 --sizes 16M,128M --algos ring:simple,tree:simple,oneshot:simple --nch 32 --iters 10 2>&1 | cut -c1-200
export POLAR_LIB=build/variants/libpolar_block.so
timeout 600 python scripts/sweep.py --n 8 --dtype f32 --sizes 16M,128M --algos ring:simple,tree:simple,oneshot:simple --nch 32 --iters 10 2>&1 | cut -c1-200
