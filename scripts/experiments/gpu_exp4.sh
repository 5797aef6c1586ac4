cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
for m in 32 128; do for c in 12 16 18; do python scripts/trace_kernel.py --mib $m --nch $c --reps 2; done; done > gpurun_out/exp4_trace.jsonl 2>&1
cat gpurun_out/exp4_trace.jsonl
