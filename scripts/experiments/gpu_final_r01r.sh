#!/bin/bash
# round-1 final evidence at HEAD: GPU tests, smoke, bench, ncu (launch list + full
# capture), BASELINE configs report, C4 latency, compute-sanitizer subset
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
bash scripts/gpu_round.sh r01r test smoke bench ncu configs c4
bash scripts/gpu_sanitize.sh
