# C4 TSQR leaf size sweep + randUTV / powerURV timelines (idle gaps per stream)
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
for ch in 0 37449 24576 16384; do
  echo "== chunk $ch" >> gpurun_out/c4_chunk.log
  timeout 600 python bench.py --workload c4 --steps 2 --warmup 1 --c4-chunk $ch >> gpurun_out/c4_chunk.log 2>&1
done
for ch in 24576 16384; do
  echo "== chunk $ch LA_CTAS=74" >> gpurun_out/c4_chunk.log
  UTV_LA_CTAS=74 timeout 600 python bench.py --workload c4 --steps 2 --warmup 1 --c4-chunk $ch >> gpurun_out/c4_chunk.log 2>&1
done
timeout 600 python tools/timeline.py rutv 16384 > gpurun_out/timeline_rutv.txt 2>&1
timeout 600 python tools/timeline.py purv 16384 > gpurun_out/timeline_purv.txt 2>&1
