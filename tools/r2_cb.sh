cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
UTV_D2H_TRACE=1 timeout 600 python tools/e2e_stages2.py > gpurun_out/e2e_trace2.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py tests/test_gpu_scale.py tests/test_gpu_spec.py -q -rfE --timeout 600 -p no:cacheprovider > gpurun_out/pytest_cb.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_cb.log
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu --no-c4 > gpurun_out/bench_cb.log 2>&1
