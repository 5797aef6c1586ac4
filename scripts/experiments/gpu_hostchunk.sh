#!/bin/bash
# e2e (polar_allreduce_host) chunk size sweep: POLAR_HOST_CHUNK bytes per rank per pipeline stage
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
for ch in 4194304 8388608 16777216 33554432; do
  POLAR_HOST_CHUNK=$ch timeout 600 python bench.py --steps 20 --warmup 3 > gpurun_out/hostchunk_$ch.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/hostchunk_$ch.json')); print($ch, d['e2e'])"
done
