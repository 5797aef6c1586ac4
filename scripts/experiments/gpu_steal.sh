#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
export POLAR_TIMEOUT_MS=5000
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "twoshot or policy or default" --timeout=600 2>&1 | tail -2
bash scripts/gpu_ab.sh nosteal
for m in 4 16 128; do timeout 300 python scripts/trace_kernel.py --n 8 --mib $m --nch 32 --reps 1; done > gpurun_out/trace_steal.jsonl 2>&1
cat gpurun_out/trace_steal.jsonl
