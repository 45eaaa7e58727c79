"""Sparsity of the slot engine's GEMM inputs (diagnostics; CPU oracle).

FISTA's second GEMM multiplies x_{k+1} (soft-thresholded) and, after the
round-2 reformulation, ADMM's first GEMM multiplies z (soft-thresholded).  A
DMMA m8n8k4 tile covers 4 coefficient rows (one k-step) of 8 slots; it can be
skipped when those 4 x 8 inputs are all zero.  This script follows every
iteration of FISTA / ADMM (lambda = 0.1) on a sample of the scaling cube's
tile 0 through the oracle, records the k-steps with a nonzero input per
pixel-iteration, and simulates the 32-slot engine (pixels refilled from a
queue as they finish) to count the DMMAs a per-8-slot-block mask and a
CTA-wide (32-slot) mask keep:

    python tools/sparsity_study.py

Measured: FISTA 0.396 (per block) vs 0.811 (CTA-wide) of the dense DMMAs of
its second GEMM; ADMM's z 0.575 vs 0.936.
"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, math
from paper_2401_14762_b200 import synth
from oracle import cpu_solvers as oc

c = synth.generate_strided('salinas', 200, workers=4)   # ~555 px
N = c.n
def track(algo, p, lam=0.1):
    a = c.basis[c.masks[p].astype(np.intp)]
    y = c.y[p]
    cfg = oc.OracleConfig(lam=lam, max_iter=5000)
    lip = oc.lipschitz(a)
    st = oc._Fista(a, y, cfg, lip) if algo == 'fista' else oc._Admm(a, y, cfg)
    masks = []
    residual = y; delta = 1.0
    while delta >= 1e-8:
        new = st(residual)
        delta = float(np.linalg.norm(new - residual)); residual = new
        v = st.x if algo == 'fista' else st.z     # GEMM-2 input (fista: x_{k+1}); admm: z (Psi z)
        ks = np.zeros(N // 4, bool)
        nz = np.flatnonzero(v)
        ks[nz // 4] = True
        masks.append(ks)
    return masks

for algo in ('fista', 'admm'):
    traj = [track(algo, p) for p in range(0, c.n_pixels, 2)]
    lens = [len(t) for t in traj]
    dens = np.concatenate([[m.mean() for m in t] for t in traj])
    print(algo, 'pixels', len(traj), 'mean iters', np.mean(lens), 'mean k-step density per pixel-iter', dens.mean())
    # slot-engine simulation: 32 slots, queue of pixels; per tick each cb of 8 slots -> union of k-steps
    rng = np.random.default_rng(0)
    order = rng.permutation(len(traj))
    q = list(order) * 4
    slots = [None] * 32
    pos = [0] * 32
    tot_dense = tot_cb = tot_cta = 0
    ticks = 0
    qi = 0
    while True:
        for s in range(32):
            if slots[s] is None or pos[s] >= len(traj[slots[s]]):
                if qi < len(q):
                    slots[s] = q[qi]; pos[s] = 0; qi += 1
                else:
                    slots[s] = None
        act = [s for s in range(32) if slots[s] is not None]
        if not act: break
        ticks += 1
        ms = [traj[slots[s]][pos[s]] if slots[s] is not None else np.zeros(N // 4, bool) for s in range(32)]
        for cb in range(4):
            u = np.zeros(N // 4, bool)
            for s in range(8 * cb, 8 * cb + 8): u |= ms[s]
            tot_cb += u.sum()
        ucta = np.zeros(N // 4, bool)
        for m in ms: ucta |= m
        tot_cta += 4 * ucta.sum()
        tot_dense += 4 * (N // 4)
        for s in act: pos[s] += 1
    print(f'  GEMM-2 DMMA fraction needed: per-cb skip {tot_cb / tot_dense:.3f}, CTA-wide skip {tot_cta / tot_dense:.3f}')
