#!/bin/bash
# A/B of the A-fragment cp.async ring (HCS_CONVEX_RING=0/1 of the current build) against variants/libhead.so:
# bitwise comparison on 100k pixels, then the bench-size launches.
out=gpurun_out/abr; mkdir -p $out
for spec in "variants/libhead.so head 1" "paper_2401_14762_b200/libhypercs_b200.so reg 0" "paper_2401_14762_b200/libhypercs_b200.so ring 1"; do
  for a in "fista 0.1 5000" "admm 0.1 5000" "fista 100 5000" "admm 100 5000" "admm 3 300"; do
    set -- $spec $a
    echo "== $2 $4 lam=$5"
    HCS_LIB=$1 HCS_CONVEX_RING=$3 python tools/run_case.py --cube salinas --algo $4 --lam $5 --cap $6 --pixels 100000 --reps 3 \
      --dump $out/$2_$4_$5.npz | tail -1
  done
done
python - "$out" <<'PY'
import sys, glob, numpy as np, os
out = sys.argv[1]
for f in sorted(glob.glob(out + "/head_*.npz")):
    c = os.path.basename(f)[5:]
    ref = np.load(f)
    for l in ("reg", "ring"):
        z = np.load(f"{out}/{l}_{c}")
        same = {k: bool(np.array_equal(ref[k], z[k], equal_nan=True)) for k in ref.files}
        print(c, l, "bitwise identical:", all(same.values()), {k: v for k, v in same.items() if not v})
PY
rm -f $out/*.npz
for r in 1; do echo "== bench-size, HCS_CONVEX_RING=$r"; HCS_CONVEX_RING=$r bash tools/ab_bench_convex.sh paper_2401_14762_b200/libhypercs_b200.so; done
