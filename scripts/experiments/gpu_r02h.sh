#!/bin/bash
# real-comm path under MPS: registered vs unregistered (bounce pipeline) at 2 bounce sizes
cd "${GRAFT_REPO_ROOT:-/root/repo}"
TAG=_b64 bash scripts/gpu_mps_bench.sh 2 4
TAG=_b256 POLAR_BOUNCE=268435456 bash scripts/gpu_mps_bench.sh 2 4
