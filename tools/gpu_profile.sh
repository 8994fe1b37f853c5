#!/bin/bash
# Full evidence run: headline bench (e2e + cpu baseline), C4/C5 benches,
# ncu launch list of a reduced bench, ncu --set full of the top kernels.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 1500 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_full.log 2>&1
timeout 900 python bench.py --workload c5 --steps 2 --warmup 1 > gpurun_out/bench_c5.log 2>&1
timeout 900 python bench.py --workload c4 --steps 2 --warmup 1 > gpurun_out/bench_c4.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --n 8192 --steps 1 --warmup 1 --no-e2e --no-cpu > gpurun_out/ncu_launch_bench.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:dgemm_tma -s 2 -c 1 -o gpurun_out/gemm_nt_r01 -f python tools/ncu_gemm.py nt > gpurun_out/ncu1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:panel_qr -s 1 -c 1 -o gpurun_out/panel16384_r01 -f python tools/ncu_small.py qr 16384 > gpurun_out/ncu2.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sgemm_tf32x3 -s 2 -c 1 -o gpurun_out/tf32_r01 -f python tools/tf32_sweep.py > gpurun_out/ncu3.log 2>&1
tail -c 600 gpurun_out/bench_full.log; tail -c 300 gpurun_out/bench_c5.log; tail -c 300 gpurun_out/bench_c4.log
