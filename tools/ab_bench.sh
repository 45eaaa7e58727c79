for spec in "variants/libhead.so 1" "paper_2401_14762_b200/libhypercs_b200.so 0" "paper_2401_14762_b200/libhypercs_b200.so 1"; do
set -- $spec
echo "== $1 DCT=$2"
HCS_LIB=$1 HCS_DCT_GRAM=$2 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e --only cosamp_k27,cosamp_k33,gomp_k27,biht_k33 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print({k:round(1777664/v*1e3,1) for k,v in d['per_solver'].items()})"
done
