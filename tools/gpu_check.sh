#!/bin/bash
# One gpurun call: GPU tests, kernel timings, bench, ncu launch list + full capture.
set -x
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python tools/quick_perf.py gemm qr svd > gpurun_out/quick_perf.log 2>&1
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/bench.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --n 8192 --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_launch_bench.log 2>&1
for s in nt tt nn; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:dgemm_tma -s 2 -c 1 -o gpurun_out/gemm_$s -f python tools/ncu_gemm.py $s > gpurun_out/ncu_gemm_$s.log 2>&1
done
timeout 300 ncu --set full --clock-control none --import-source on -k regex:leaf_qr -s 20 -c 1 -o gpurun_out/leafqr -f python tools/ncu_small.py qr > gpurun_out/ncu_qr.log 2>&1
