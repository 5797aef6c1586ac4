cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
export POLAR_TIMEOUT_MS=5000
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout=600 > gpurun_out/pytest_exp8.log 2>&1; tail -2 gpurun_out/pytest_exp8.log
for n in 2 4 8; do for dt in f32 bf16; do python scripts/sweep.py --n $n --dtype $dt --sizes 16M,128M,512M --algos twoshot:simple --nch 16,32 --iters 10 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        r=json.loads(l); print(r['n'], r['dtype'], r['bytes']>>20, r['nch'], r.get('us'), r.get('busbw_gbs'), r.get('min_hbm_gbs'))
    else: print(l.strip()[:200])
"; done; done
python bench.py --steps 50 | cut -c1-250
