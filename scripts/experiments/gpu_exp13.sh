cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
export POLAR_TIMEOUT_MS=5000
timeout 900 python -m pytest tests/test_gpu_collectives.py tests/test_gpu_graphs.py -q -x --timeout=600 2>&1 | tail -2
python scripts/report_configs.py --configs f4 | python -c "
import sys,json
for l in sys.stdin:
    r=json.loads(l)
    if 'bytes' in r: print(r['bytes']>>10,'KiB', {k:v['busbw_gbs'] for k,v in r.items() if isinstance(v,dict)})"
