cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
export POLAR_TIMEOUT_MS=5000
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout=600 > gpurun_out/pytest_exp3.log 2>&1; tail -2 gpurun_out/pytest_exp3.log
for v in u1 u2 u2lb1 u4lb1; do
  POLAR_LIB=build/variants/libpolar_$v.so timeout 300 python scripts/sweep.py --n 8 --sizes 32M,128M --algos twoshot:simple --nch 12,14,16,18,24,32 --iters 30 > gpurun_out/exp3_$v.jsonl 2>&1
  echo "== $v"; python -c "
import json
for l in open('gpurun_out/exp3_$v.jsonl'):
    if l.startswith('{'):
        r=json.loads(l); print(r['bytes']>>20, r['nch'], r.get('us'), r.get('min_hbm_gbs'))
    else: print(l.strip()[:200])
"
done
