# A/B on the bench's full cube: tools/ab_bench.sh "lib env=val" ... [-- solver,labels]
only=${ONLY:-cosamp_k27,cosamp_k33,gomp_k27,biht_k33}
for spec in "$@"; do
set -- $spec
echo "== $spec"
env HCS_LIB=$1 $2 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --only $only 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print({k:round(1777664/v*1e3,1) for k,v in d['per_solver'].items()})"
done
