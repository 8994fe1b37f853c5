cd "${GRAFT_REPO_ROOT:-.}"
for w in gemm qr svd qrcp rutv purv purv_overlap; do
  echo "== san_$w"; timeout 900 compute-sanitizer --tool memcheck python tools/sanitize_small.py $w 2>&1 | tail -2
done
UTV_QRCP_BIG=1 bash -c 'echo "== san_qrcp_big"; timeout 900 compute-sanitizer --tool memcheck python tools/sanitize_small.py qrcp 2>&1 | tail -2'
for w in svd qr gemm qrcp; do
  echo "== race_$w"; timeout 900 compute-sanitizer --tool racecheck python tools/sanitize_small.py $w 2>&1 | tail -2
done
