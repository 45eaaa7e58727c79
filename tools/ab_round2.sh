#!/bin/bash
# A/B of the round-2 greedy changes against the committed HEAD build (100k... 40k salinas pixels):
#   variants/libhead.so          HEAD
#   current, HCS_DCT_GRAM=0      warp-gOMP 16-row groups + batched L2 loads in the refinement / residual
#   current                      + DCT closed-form Gram
out=gpurun_out/ab2; mkdir -p $out
cp paper_2401_14762_b200/libhypercs_b200.so variants/libnew.so
for spec in "variants/libhead.so head 1" "variants/libnew.so nodct 0" "variants/libnew.so new 1"; do
  set -- $spec
  echo "== $2 ($1, HCS_DCT_GRAM=$3)"
  for a in "gomp 27" "gomp 33" "biht 27" "biht 33" "cosamp 27" "cosamp 33"; do
    set -- $spec $a
    HCS_LIB=$1 HCS_DCT_GRAM=$3 python tools/run_case.py --cube salinas --algo $4 --kappa $5 --pixels 100000 --reps 3 \
      --dump $out/$2_$4$5.npz | tail -1
  done
done
python - "$out" <<'PY'
import sys, glob, numpy as np, os
out = sys.argv[1]
for c in sorted({os.path.basename(f).split("_", 1)[1] for f in glob.glob(out + "/*.npz")}):
    ref = np.load(f"{out}/head_{c}")
    for l in ("nodct", "new"):
        z = np.load(f"{out}/{l}_{c}")
        same = all(np.array_equal(ref[k], z[k]) for k in ref.files)
        msg = f"{c}: {l} vs head bitwise identical: {same}"
        if not same:
            nr = np.maximum(np.linalg.norm(ref["x"], axis=1), 1e-300)
            rel = np.linalg.norm(ref["x"] - z["x"], axis=1) / nr
            itd = ref["iterations"] != z["iterations"]
            msg += (f"; iteration mismatches {int(itd.sum())}, converged mismatches "
                    f"{int((ref['converged'] != z['converged']).sum())}, max rel dx (equal-iteration pixels) "
                    f"{rel[~itd].max():.2e}, pixels with rel dx > 1e-9: {int((rel[~itd] > 1e-9).sum())}")
        print(msg)
PY
rm -f $out/*.npz
echo "== phases (variants/libnewph.so, -DHCS_PHASES; DCT Gram on, then off)"
for g in 1 0; do
for a in "biht 27" "cosamp 27" "cosamp 33"; do
  set -- $a
  HCS_LIB=variants/libnewph.so HCS_DCT_GRAM=$g python tools/run_case.py --cube salinas --algo $1 --kappa $2 --pixels 40000 --reps 2 | tail -4
done
done
