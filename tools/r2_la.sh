# look-ahead panel budget / adaptive full-width panels: C2 and the headline powerURV
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
for env in "UTV_LA_CTAS=48 UTV_LA_ADAPT=0" "UTV_LA_CTAS=32 UTV_LA_ADAPT=0" "UTV_LA_CTAS=64 UTV_LA_ADAPT=0" \
           "UTV_LA_CTAS=48 UTV_LA_ADAPT=2048" "UTV_LA_CTAS=48 UTV_LA_ADAPT=4096" "UTV_LA_CTAS=64 UTV_LA_ADAPT=2048"; do
  echo "== $env" >> gpurun_out/la_c2.log
  env $env timeout 300 python bench.py --workload c2 --steps 3 --warmup 2 >> gpurun_out/la_c2.log 2>&1
  echo "== $env" >> gpurun_out/la_head.log
  env $env timeout 600 python bench.py --steps 2 --warmup 2 --no-e2e --no-cpu --no-c4 >> gpurun_out/la_head.log 2>&1
done
