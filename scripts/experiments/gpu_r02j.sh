#!/bin/bash
# round-2 evidence: sanitizers (incl. TMA ring), per-config report, C4 latency
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
bash scripts/gpu_sanitize.sh
timeout 2400 python scripts/report_configs.py > gpurun_out/configs_r02j.jsonl 2> gpurun_out/configs_r02j.err; echo "configs rc=$?"
timeout 900 python scripts/c4_latency.py > gpurun_out/c4_r02j.jsonl 2>&1; echo "c4 rc=$?"
