cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
export POLAR_TIMEOUT_MS=5000
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout=600 > gpurun_out/pytest_exp5.log 2>&1; tail -2 gpurun_out/pytest_exp5.log
for v in lb1 lb2; do
  echo "== $v"
  for m in 32 128; do for c in 12 16 18; do POLAR_LIB=build/variants/libpolar_$v.so python scripts/trace_kernel.py --mib $m --nch $c --reps 1; done; done
  POLAR_LIB=build/variants/libpolar_$v.so timeout 300 python scripts/sweep.py --n 8 --sizes 4M,16M,32M,64M,128M --algos twoshot:simple --nch 12,16,18 --iters 30 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        r=json.loads(l); print(r['bytes']>>20, r['nch'], r.get('us'), r.get('min_hbm_gbs'))
    else: print(l.strip()[:200])
"
done
