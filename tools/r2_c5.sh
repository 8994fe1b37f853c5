cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 900 python bench.py --workload c5 --steps 2 --warmup 2 > gpurun_out/bench_c5.log 2>&1
timeout 900 python bench.py --workload c2 --steps 3 --warmup 3 > gpurun_out/bench_c2.log 2>&1
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1
