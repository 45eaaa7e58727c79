#!/bin/bash
# A/B of the skewed ADMM schedule (HCS_CONVEX_SKEW=0/1, lead variants) against variants/libhead.so
out=gpurun_out/abs; mkdir -p $out
for spec in "variants/libhead.so head 1" "paper_2401_14762_b200/libhypercs_b200.so noskew 0" "paper_2401_14762_b200/libhypercs_b200.so skew 1"; do
  for a in "admm 0.1 5000" "admm 100 5000" "admm 3 300" "admm 1 300"; do
    set -- $spec $a
    echo "== $2 $4 lam=$5"
    HCS_LIB=$1 HCS_CONVEX_SKEW=$3 python tools/run_case.py --cube salinas --algo $4 --lam $5 --cap $6 --pixels 100000 --reps 3 \
      --dump $out/$2_$4_$5.npz | tail -1
  done
done
python - "$out" <<'PY'
import sys, glob, numpy as np, os
out = sys.argv[1]
for f in sorted(glob.glob(out + "/head_*.npz")):
    c = os.path.basename(f)[5:]
    ref = np.load(f)
    for l in ("noskew", "skew"):
        z = np.load(f"{out}/{l}_{c}")
        same = {k: bool(np.array_equal(ref[k], z[k], equal_nan=True)) for k in ref.files}
        print(c, l, "bitwise identical:", all(same.values()), {k: v for k, v in same.items() if not v})
PY
rm -f $out/*.npz
bench1() { HCS_LIB=$1 HCS_CONVEX_SKEW=$2 python bench.py --steps 3 --warmup 1 --no-e2e --no-cpu --only admm_l0.1 2>/dev/null | python -c "
import sys, json
d = json.loads(sys.stdin.readlines()[-1]); print(d['ms_per_step'], d['roofline'].get('frac'))"; }
echo "== bench-size admm_l0.1: noskew, skew (lead 2), lead 0, 4, 8"
bench1 paper_2401_14762_b200/libhypercs_b200.so 0
bench1 paper_2401_14762_b200/libhypercs_b200.so 1
for l in 0 4 8; do bench1 variants/liblead$l.so 1; done
