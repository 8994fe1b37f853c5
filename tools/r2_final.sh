# full GPU suite + smoke + default bench + C4/C5 lines + ncu launch list
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -rfE --timeout 900 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1200 python bench.py > gpurun_out/bench_default.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_default.log
timeout 900 python bench.py --workload c4 --steps 2 --warmup 1 > gpurun_out/bench_c4.log 2>&1
timeout 900 python bench.py --workload c5 --steps 2 --warmup 1 > gpurun_out/bench_c5.log 2>&1
timeout 900 python bench.py --workload c2 --steps 3 --warmup 3 > gpurun_out/bench_c2.log 2>&1
