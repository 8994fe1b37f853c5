# full GPU suite + smoke + tstore0 A/B on top of the per-warp stores
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -rfE --timeout 900 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
for env in "UTV_GEMM_TSTORE0=1" "UTV_GEMM_TSTORE0=0"; do
  env $env timeout 300 python tools/gemm_ab.py >> gpurun_out/gemm_ab_t0.log 2>&1
  echo "== $env" >> gpurun_out/bench_t0.log
  env $env timeout 600 python bench.py --steps 2 --warmup 2 --no-e2e --no-cpu --no-c4 >> gpurun_out/bench_t0.log 2>&1
done
