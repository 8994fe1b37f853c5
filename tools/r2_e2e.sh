cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 300 python tools/d2h_bench.py > gpurun_out/d2h_bench.log 2>&1
timeout 600 python tools/e2e_stages2.py > gpurun_out/e2e_stages2.log 2>&1
