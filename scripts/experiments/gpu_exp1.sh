cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
export POLAR_TIMEOUT_MS=5000
timeout 600 python -m pytest tests -m gpu -q -x --timeout=600 > gpurun_out/pytest_exp1.log 2>&1; tail -2 gpurun_out/pytest_exp1.log
python scripts/sweep.py --n 8 --sizes 32M,128M --algos twoshot:simple --nch 8,12,14,16,18 > gpurun_out/exp1_ts.jsonl 2>&1
python scripts/sweep.py --n 8 --sizes 8,256,4K,32K,256K --algos oneshot:ll,oneshot:simple,twoshot:ll,twoshot:simple,tree:ll,ring:ll --nch 1,2,4 --graph > gpurun_out/exp1_small_graph.jsonl 2>&1
python scripts/sweep.py --n 8 --sizes 8,4K,256K --algos oneshot:ll,twoshot:simple --nch 1,4 > gpurun_out/exp1_small_eager.jsonl 2>&1
cat gpurun_out/exp1_ts.jsonl
