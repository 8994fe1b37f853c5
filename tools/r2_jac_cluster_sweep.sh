cd $GRAFT_REPO_ROOT
for c in 2 4 8; do
  UTV_JAC_CLUSTER=$c timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-c4 2>/dev/null | grep '^{' | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('C=$c', d['ms_per_step'], d['seconds'], d['kernels']['jacobi'])"
done
