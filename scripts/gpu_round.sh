#!/bin/bash
# GPU session: parity tests, smoke, bench, ncu launch list + one full capture
# usage: bash scripts/gpu_round.sh [tag] [what...]   what in {test,smoke,bench,ncu,configs,c4,tune,sweep}
cd "${GRAFT_REPO_ROOT:-/root/repo}"
TAG=${1:-r01}; shift
WHAT=${@:-test smoke bench ncu}
mkdir -p gpurun_out
export POLAR_TIMEOUT_MS=${POLAR_TIMEOUT_MS:-5000}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,temperature.gpu --format=csv > gpurun_out/nvsmi_$TAG.txt 2>&1
for w in $WHAT; do
  case $w in
    test)
      timeout 1800 python -m pytest tests -m gpu -q -rf --timeout=600 > gpurun_out/pytest_gpu_$TAG.log 2>&1
      echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$TAG.log; tail -4 gpurun_out/pytest_gpu_$TAG.log ;;
    smoke)
      timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke_$TAG.log 2>&1
      echo "smoke rc=$?" >> gpurun_out/smoke_$TAG.log; tail -2 gpurun_out/smoke_$TAG.log ;;
    bench)
      timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
      echo "bench rc=$?"; cat gpurun_out/bench_$TAG.json | cut -c1-600 ;;
    ncu)
      timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
        --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 20 --warmup 3 > gpurun_out/ncu_launch_bench_$TAG.log 2>&1
      echo "ncu launches rc=$?"
      # the timed region only (NVTX range "timed" in bench.py): the step's kernels and their shares
      timeout 900 ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum --clock-control none --csv \
        --log-file gpurun_out/launches_timed_$TAG.csv python bench.py --steps 20 --warmup 3 > gpurun_out/ncu_launch_timed_$TAG.log 2>&1
      echo "ncu timed launches rc=$?"
      timeout 1200 ncu --set full --clock-control none --import-source on -k regex:allreduce_kernel -s 5 -c 1 \
        -f -o gpurun_out/prof_$TAG python bench.py --steps 8 --warmup 3 > gpurun_out/ncu_full_$TAG.log 2>&1
      echo "ncu full rc=$?" ;;
    configs)
      timeout 2400 python scripts/report_configs.py > gpurun_out/configs_$TAG.jsonl 2> gpurun_out/configs_$TAG.err
      echo "configs rc=$?"; tail -3 gpurun_out/configs_$TAG.jsonl | cut -c1-300 ;;
    c4)
      timeout 900 python scripts/c4_latency.py > gpurun_out/c4_$TAG.jsonl 2>&1; echo "c4 rc=$?" ;;
    tune)
      timeout 1800 python scripts/tune_policy.py --n 2,4,8 > gpurun_out/tune_$TAG.jsonl 2> gpurun_out/tune_$TAG.err
      echo "tune rc=$?"; grep table gpurun_out/tune_$TAG.jsonl | cut -c1-300 ;;
    sweep)
      timeout 900 python scripts/sweep.py --n 8 --dtype f32 > gpurun_out/sweep_f32_$TAG.jsonl 2>&1
      echo "sweep rc=$?" ;;
  esac
done
