cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
export POLAR_TIMEOUT_MS=5000
timeout 900 python -m pytest tests/test_gpu_multiproc.py -q -x --timeout=900 > gpurun_out/pytest_mp_exp2.log 2>&1; tail -3 gpurun_out/pytest_mp_exp2.log
for v in u1lb2 u2lb1 u1lb1 b1024 b256 b256u2; do
  POLAR_LIB=build/variants/libpolar_$v.so timeout 300 python scripts/sweep.py --n 8 --sizes 128M --algos twoshot:simple --nch 8,12,14,16,18,24,32 --iters 30 > gpurun_out/exp2_$v.jsonl 2>&1
  echo "== $v"; python -c "
import json,sys
for l in open('gpurun_out/exp2_$v.jsonl'):
    if l.startswith('{'):
        r=json.loads(l); print(r['nch'], r.get('us'), r.get('min_hbm_gbs'))
    else: print(l.strip()[:200])
"
done
