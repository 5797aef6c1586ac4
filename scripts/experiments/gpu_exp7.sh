cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
export POLAR_TIMEOUT_MS=5000
timeout 900 python -m pytest tests -m gpu -q -x --timeout=600 > gpurun_out/pytest_exp7.log 2>&1; tail -2 gpurun_out/pytest_exp7.log
for pdl in 1 0; do echo "== PDL=$pdl"; POLAR_PDL=$pdl python scripts/trace_kernel.py --mib 128 --nch 16 --reps 1; POLAR_PDL=$pdl python scripts/trace_kernel.py --mib 4 --nch 16 --reps 1
POLAR_PDL=$pdl python bench.py --steps 100 --warmup 5 | cut -c1-300; done
timeout 900 python scripts/c4_latency.py > gpurun_out/c4_latency.jsonl 2>&1; echo "c4 rc=$?"; tail -3 gpurun_out/c4_latency.jsonl
