#!/bin/bash
# round 2: new parity tests (C2 size multi-process, C3 1 GiB n=4, n=4 matrix), bench N=1 line
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
export POLAR_TIMEOUT_MS=${POLAR_TIMEOUT_MS:-20000}
timeout 600 python -m pytest tests/test_gpu_multiproc.py -q -x -k north_star -s > gpurun_out/r02b_c2.log 2>&1; echo "c2 rc=$?"; tail -5 gpurun_out/r02b_c2.log
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "c3_bf16 or matrix_sum" > gpurun_out/r02b_parity.log 2>&1; echo "parity rc=$?"; tail -3 gpurun_out/r02b_parity.log
timeout 900 python -m pytest tests/test_gpu_bench.py tests/test_gpu_collectives.py -q -x > gpurun_out/r02b_bench_tests.log 2>&1; echo "bench tests rc=$?"; tail -3 gpurun_out/r02b_bench_tests.log
timeout 600 python bench.py > gpurun_out/r02b_bench.json 2> gpurun_out/r02b_bench.err; echo "bench rc=$?"; cut -c1-400 gpurun_out/r02b_bench.json
