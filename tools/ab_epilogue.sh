#!/bin/bash
# A/B of the round-2 convex epilogues (column-block staged loads, thread-order row map, branch-free
# soft-threshold division) against variants/libhead.so: tools/ab_epilogue.sh [pixels]
out=gpurun_out/abe; mkdir -p $out
px=${1:-100000}
python - <<'PY'
import ctypes
from paper_2401_14762_b200 import _native
lib = _native.load()
lib.hcs_debug_divcheck.argtypes = [ctypes.c_ulonglong, ctypes.c_ulonglong, ctypes.c_int, ctypes.POINTER(ctypes.c_ulonglong)]
for mode in (0, 1, 2):
    o = (ctypes.c_ulonglong * 3)()
    rc = lib.hcs_debug_divcheck(1 << 32, 12345 + mode, mode, o)
    print(f"divcheck mode {mode}: rc {rc}, accepted {o[0]}, accepted-but-different {o[1]}, rejected {o[2]}")
PY
for spec in "variants/libhead.so head" "paper_2401_14762_b200/libhypercs_b200.so new"; do
  set -- $spec
  for a in "fista 0.1 5000" "admm 0.1 5000" "fista 100 5000" "admm 100 5000" "admm 3 300"; do
    set -- $spec $a
    echo "== $2 $3 lam=$4"
    HCS_LIB=$1 python tools/run_case.py --cube salinas --algo $3 --lam $4 --cap $5 --pixels $px --reps 3 \
      --dump $out/$2_$3_$4.npz | tail -2
  done
done
python - "$out" <<'PY'
import sys, glob, numpy as np, os
out = sys.argv[1]
for f in sorted(glob.glob(out + "/head_*.npz")):
    c = os.path.basename(f)[5:]
    ref, z = np.load(f), np.load(f"{out}/new_{c}")
    same = {k: bool(np.array_equal(ref[k], z[k], equal_nan=True)) for k in ref.files}
    print(c, "bitwise identical:", all(same.values()), {k: v for k, v in same.items() if not v})
PY
rm -f $out/*.npz
echo "== phases head / new (fista, admm lam 0.1)"
for l in variants/libheadph.so variants/libnewph.so; do for a in fista admm; do
HCS_LIB=$l python tools/run_case.py --cube salinas --algo $a --lam 0.1 --cap 5000 --pixels 40000 --reps 2 | tail -3
done; done
