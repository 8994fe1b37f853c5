# A/B: QR / apply group widths, fused split-K and the beta=0 staged epilogue on
# the headline step; GEMM epilogue variants; re-run of the fixed tests.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_spec.py tests/test_gpu_parity.py -q -rfE --timeout 600 -p no:cacheprovider -k "ragged or acceptance" > gpurun_out/pytest_fix.log 2>&1
for env in "UTV_QR_GROUP=256 UTV_APPLY_GROUP=256 UTV_SPLITK_FUSE_MAX=0" \
           "UTV_QR_GROUP=512 UTV_APPLY_GROUP=512 UTV_SPLITK_FUSE_MAX=4" \
           "UTV_QR_GROUP=256 UTV_APPLY_GROUP=512 UTV_SPLITK_FUSE_MAX=4" \
           "UTV_QR_GROUP=512 UTV_APPLY_GROUP=256 UTV_SPLITK_FUSE_MAX=4" \
           "UTV_QR_GROUP=256 UTV_APPLY_GROUP=256 UTV_SPLITK_FUSE_MAX=4" \
           "UTV_QR_GROUP=256 UTV_APPLY_GROUP=256 UTV_SPLITK_FUSE_MAX=0 UTV_GEMM_TSTORE0=1"; do
  echo "== $env" >> gpurun_out/bench_ab.log
  env $env timeout 600 python bench.py --steps 2 --warmup 2 --no-e2e --no-cpu --no-c4 >> gpurun_out/bench_ab.log 2>&1
done
for env in "UTV_GEMM_TSTORE0=0 UTV_SPLITK_FUSE_MAX=0" "UTV_GEMM_TSTORE0=1 UTV_SPLITK_FUSE_MAX=4"; do
  env $env timeout 300 python tools/gemm_ab.py >> gpurun_out/gemm_ab.log 2>&1
done
