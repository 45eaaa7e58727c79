#!/bin/bash
# bench-size A/B (1.78M px) of the convex launches: tools/ab_bench_convex.sh LIB...
for l in "$@"; do for c in admm_l0.1 fista_l0.1; do
echo "== $l $c"
HCS_LIB=$l python bench.py --steps 3 --warmup 1 --no-e2e --no-cpu --only $c 2>/dev/null | python -c "
import sys, json
d = json.loads(sys.stdin.readlines()[-1]); print(d['ms_per_step'], d['roofline'].get('frac'), d['clocks'])"
done; done
