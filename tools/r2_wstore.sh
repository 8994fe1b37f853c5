# per-warp TMA-store epilogue: correctness (GEMM tests, out-of-view sweep) and A/B
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py -q -rfE --timeout 600 -p no:cacheprovider > gpurun_out/pytest_wstore.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_wstore.log
timeout 600 python tools/gemm_oob_sweep.py > gpurun_out/oob_sweep.log 2>&1; echo "rc=$?" >> gpurun_out/oob_sweep.log
for env in "UTV_GEMM_WSTORE=0" "UTV_GEMM_WSTORE=1"; do
  env $env timeout 300 python tools/gemm_ab.py >> gpurun_out/gemm_ab_ws.log 2>&1
  echo "== $env" >> gpurun_out/bench_ws.log
  env $env timeout 600 python bench.py --steps 2 --warmup 2 --no-e2e --no-cpu --no-c4 >> gpurun_out/bench_ws.log 2>&1
done
