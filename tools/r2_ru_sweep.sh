# randUTV side-stream / panel CTA budgets after the Gram-form Jacobi (32-CTA clusters)
cd "${GRAFT_REPO_ROOT:-.}"
for cfg in "88 48" "64 48" "104 48" "88 32" "88 64" "72 40"; do
  set -- $cfg
  r=$(UTV_RU_SIDE=$1 UTV_RU_PANEL=$2 timeout 900 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-c4 2>/dev/null | grep '^{' | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['seconds']['randutv'], d['ms_per_step'], d['clocks']['sm_mhz'])")
  echo "UTV_RU_SIDE=$1 UTV_RU_PANEL=$2 randutv/step/mhz $r"
done
