cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
UTV_D2H_TRACE=1 timeout 600 python tools/e2e_stages2.py > gpurun_out/e2e_trace.log 2>&1
