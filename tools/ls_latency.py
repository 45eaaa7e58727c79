"""Latency (P=1) and throughput (P=many) of the batched least-squares kernel."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
from paper_2401_14762_b200 import kernels, synth

import ctypes
from paper_2401_14762_b200 import _native
LIB = _native.load()
PH = (ctypes.c_ulonglong * 16)()
HAS_PH = LIB.hcs_debug_phases_ls(PH, 1) == 0
NAMES = {3: "gather", 4: "gram", 11: "diag0", 12: "panels", 13: "trail+diag", 5: "chol-end", 6: "solve+refine",
         10: "out"}


def run(M, K, P, reps=5):
    rng = np.random.default_rng(0)
    basis = synth.dct_basis(224)
    b = np.empty((P, M, K)); y = np.empty((P, M))
    for p in range(P):
        rows = np.sort(rng.choice(224, M, replace=False)); cols = np.sort(rng.choice(224, K, replace=False))
        b[p] = basis[np.ix_(rows, cols)]; y[p] = rng.standard_normal(M)
    bd = torch.as_tensor(b, device="cuda"); yd = torch.as_tensor(y, device="cuda")
    kernels.least_squares(bd, yd)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(reps):
        e0.record(); s, path = kernels.least_squares(bd, yd, return_path=True); e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) * 1e3)
    if HAS_PH:
        LIB.hcs_debug_phases_ls(PH, 1)
        kernels.least_squares(bd, yd)
        torch.cuda.synchronize()
        LIB.hcs_debug_phases_ls(PH, 1)
        print("   cycles/system: " + ", ".join(f"{nm} {PH[i] / P:.0f}" for i, nm in NAMES.items()))
    ref = np.linalg.lstsq(b[0], y[0], rcond=None)[0]
    err = np.linalg.norm(s[0].cpu().numpy() - ref) / np.linalg.norm(ref)
    print(f"LS M={M} K={K} P={P}: {best:.1f} us total, {best / P:.2f} us/system, path0={int((path == 0).sum())}/{P}, rel err {err:.1e}")

for K in (8, 27, 54, 81, 90):
    run(90, K, 1)
for K in (27, 81):
    run(90, K, 296 * 4)
