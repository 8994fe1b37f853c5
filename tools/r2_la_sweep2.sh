cd "${GRAFT_REPO_ROOT:-.}"
for la in 64 96 128; do
  c2=$(UTV_LA_CTAS=$la timeout 600 python bench.py --workload c2 --steps 3 --warmup 3 2>/dev/null | grep '^{' | python -c "import json,sys; print(json.loads(sys.stdin.read())['ms_per_step'])")
  hd=$(UTV_LA_CTAS=$la timeout 900 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-c4 2>/dev/null | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['seconds']['powerurv'])")
  echo "UTV_LA_CTAS=$la C2 $c2 headline $hd"
done
