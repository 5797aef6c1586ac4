#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
export POLAR_TIMEOUT_MS=10000
timeout 600 python scripts/experiments/exp_ring_tma.py > gpurun_out/r02c_ring_tma_ab.jsonl 2> gpurun_out/r02c_ring_tma_ab.err; echo "ab rc=$?"
cat gpurun_out/r02c_ring_tma_ab.jsonl | cut -c1-220; tail -5 gpurun_out/r02c_ring_tma_ab.err
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "ring" > gpurun_out/r02c_parity_ring.log 2>&1; echo "parity rc=$?"; tail -3 gpurun_out/r02c_parity_ring.log
timeout 600 python -m pytest tests/test_gpu_bench.py -q -x > gpurun_out/r02c_bench_tests.log 2>&1; echo "bench tests rc=$?"; tail -3 gpurun_out/r02c_bench_tests.log
