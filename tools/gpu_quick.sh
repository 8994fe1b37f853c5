#!/bin/bash
# Usage (under gpurun): bash tools/gpu_quick.sh "<pytest -k expr or 'all' or 'none'>" [bench] [perf]
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
K="$1"; shift
if [ "$K" = "all" ]; then timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log; tail -3 gpurun_out/pytest_gpu.log
elif [ "$K" != "none" ]; then timeout 900 python -m pytest tests -m gpu -x -q -k "$K" > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log; tail -3 gpurun_out/pytest_gpu.log; fi
for a in "$@"; do
  case $a in
    bench) timeout 900 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/bench.log 2>&1; tail -c 1500 gpurun_out/bench.log;;
    benchfull) timeout 1200 python bench.py --steps 3 --warmup 3 > gpurun_out/bench.log 2>&1; tail -c 3000 gpurun_out/bench.log;;
    perf*) timeout 600 python tools/quick_perf.py ${a#perf} > gpurun_out/quick_perf.log 2>&1; grep -v '^ \|^{\|^}' gpurun_out/quick_perf.log | head -40;;
  esac
done
