#!/bin/bash
# (1) GPU tests at HEAD (two-shot LL staging 256 KiB); (2) A/B two-shot generic
# path U=2 packs per rank in flight (n >= 5) vs U=1; (3) ring Simple DRAM bytes (no discard)
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
export POLAR_TIMEOUT_MS=5000
timeout 1500 python -m pytest tests -m gpu -q -x --timeout=600 > gpurun_out/ugen_pytest.log 2>&1; tail -2 gpurun_out/ugen_pytest.log
bash scripts/gpu_ab.sh ugen2
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:allreduce_kernel -c 3 --csv \
  python scripts/sweep.py --n 8 --dtype f32 --sizes 128M --algos ring:simple --nch 18 --iters 1 --warm 1 > gpurun_out/ring_dram_ncu.csv 2>&1
grep -E "dram__bytes|gpu__time" gpurun_out/ring_dram_ncu.csv | awk -F'","' '{print $13, $15}'
