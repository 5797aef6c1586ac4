#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 300 python scripts/probe_ll128.py > gpurun_out/probe_ll128.jsonl 2>&1; echo "probe rc=$?"; cat gpurun_out/probe_ll128.jsonl
