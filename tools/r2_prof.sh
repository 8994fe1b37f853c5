# ragged parity detail, default bench, ncu launch list (n=8192) and one full
# capture of the dominant GEMM launch.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -rfE --timeout 600 -p no:cacheprovider -k "ragged" > gpurun_out/pytest_ragged.log 2>&1
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/bench.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r02.csv python bench.py --n 8192 --steps 1 --warmup 1 --no-e2e --no-cpu --no-c4 > gpurun_out/ncu_launch_bench.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:dgemm_tma -s 2 -c 1 -o gpurun_out/r02_gemm_nt -f python tools/ncu_gemm.py nt > gpurun_out/ncu_gemm_nt.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:panel_qr -s 1 -c 1 -o gpurun_out/r02_panel -f python tools/ncu_small.py qr > gpurun_out/ncu_panel.log 2>&1
