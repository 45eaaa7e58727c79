#!/bin/bash
# A/B of library variants on the greedy configurations with bitwise comparison of the results
#   tools/ab_dump.sh OUTDIR lib ...     (the first lib is the reference for the comparison)
out=$1; shift
mkdir -p $out
for lib in "$@"; do
  n=$(basename $lib .so)
  echo "== $lib"
  for a in "gomp 27" "gomp 33" "biht 27" "biht 33" "cosamp 27" "cosamp 33"; do
    set -- $a
    HCS_LIB=$lib python tools/run_case.py --cube salinas --algo $1 --kappa $2 --pixels 40000 --reps 3 \
      --dump $out/${n}_$1$2.npz | tail -1
  done
done
python - "$out" <<'PY'
import sys, glob, numpy as np, os
out = sys.argv[1]
files = sorted(glob.glob(out + "/*.npz"))
libs = sorted({os.path.basename(f).split("_")[0] for f in files})
cases = sorted({os.path.basename(f).split("_", 1)[1] for f in files})
for c in cases:
    ref = np.load(f"{out}/{libs[0]}_{c}")
    for l in libs[1:]:
        z = np.load(f"{out}/{l}_{c}")
        same = all(np.array_equal(ref[k], z[k]) for k in ref.files)
        msg = f"{c}: {l} vs {libs[0]} bitwise identical: {same}"
        if not same:
            nr = np.maximum(np.linalg.norm(ref["x"], axis=1), 1e-300)
            rel = np.linalg.norm(ref["x"] - z["x"], axis=1) / nr
            itd = ref["iterations"] != z["iterations"]
            msg += (f"; iteration mismatches {int(itd.sum())}, converged mismatches "
                    f"{int((ref['converged'] != z['converged']).sum())}, max rel dx over equal-iteration pixels "
                    f"{rel[~itd].max():.2e}, pixels with rel dx > 1e-9: {int((rel[~itd] > 1e-9).sum())}")
        print(msg)
PY
