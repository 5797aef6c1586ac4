cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
for rep in 1 2 3; do for tma in 0 1; do
  POLAR_TWOSHOT_TMA=$tma python bench.py --steps 300 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('tma=$tma', d['value'], d['ms_per_step'], d['roofline']['frac'], d['clocks']['sm_mhz'], d['c2_sweep']['134217728']['us'], d['c2_sweep']['4194304']['us'], d['c2_sweep']['33554432']['us'])"
done; done
