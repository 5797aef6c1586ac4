cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
export POLAR_TIMEOUT_MS=5000
POLAR_TWOSHOT_TMA=1 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout=600 -k "twoshot or policy or bench_size or back_to_back" > gpurun_out/pytest_exp11.log 2>&1; tail -2 gpurun_out/pytest_exp11.log
for n in 2 4 8; do POLAR_TWOSHOT_TMA=1 python scripts/sweep.py --n $n --dtype f32 --sizes 1M,16M,128M,512M --algos twoshot:simple --nch 16,32 --iters 10 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        r=json.loads(l); print('tma', r['n'], r['bytes']>>20, r['nch'], r.get('us'), r.get('busbw_gbs'), r.get('min_hbm_gbs'))
    else: print(l.strip()[:300])
"; done
POLAR_TWOSHOT_TMA=1 python scripts/trace_kernel.py --mib 128 --nch 32 --reps 1
