cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py tests/test_gpu_scale.py -q -rfE --timeout 600 -p no:cacheprovider > gpurun_out/pytest_cols.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_cols.log
timeout 600 python tools/e2e_stages2.py > gpurun_out/e2e_stages2b.log 2>&1
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu --no-c4 > gpurun_out/bench_cols.log 2>&1
