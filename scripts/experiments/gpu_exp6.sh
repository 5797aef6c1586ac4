cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
for coop in 1 0; do
  echo "== coop=$coop"
  for m in 0.0625 4 128; do POLAR_VIRTUAL_COOP=$coop python scripts/trace_kernel.py --mib $m --nch 16 --reps 1; done
  POLAR_VIRTUAL_COOP=$coop timeout 300 python scripts/sweep.py --n 8 --sizes 64K,4M,32M,128M --algos twoshot:simple,oneshot:simple --nch 16 --iters 30 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        r=json.loads(l); print(r['bytes']>>10,'KiB', r['algo'], r['nch'], r.get('us'), r.get('min_hbm_gbs'))
    else: print(l.strip()[:200])
"
done
python bench.py --steps 50 --warmup 5 | cut -c1-400
