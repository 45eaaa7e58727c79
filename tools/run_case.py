"""Run one solver configuration on a synthetic cube slice (profiling helper).

    python tools/run_case.py --cube salinas --algo cosamp --kappa 27 --pixels 8000 [--reps 3]
"""

import argparse
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2401_14762_b200 import synth  # noqa: E402
from paper_2401_14762_b200.solvers import SolverConfig, solve_batch  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cube", default="salinas")
    ap.add_argument("--algo", default="cosamp")
    ap.add_argument("--kappa", type=int, default=27)
    ap.add_argument("--lam", type=float, default=0.1)
    ap.add_argument("--cap", type=int, default=2000)
    ap.add_argument("--pixels", type=int, default=8000)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--dump", default=None, help="save x / iterations / flags of the last rep (.npz)")
    args = ap.parse_args()
    n = synth.CUBES[args.cube]["n"]
    rows = max(1, args.pixels // 100)
    cube = synth.generate(rows, 100, n, seed=11)
    dev = torch.device("cuda")
    y = torch.as_tensor(cube.y, device=dev)
    m = torch.as_tensor(cube.masks, device=dev)
    b = torch.as_tensor(cube.basis, device=dev)
    params = dict(kappa=args.kappa) if args.algo in ("gomp", "biht", "cosamp") else dict(lam=args.lam)
    cfg = SolverConfig(time_limit=None, max_iter=args.cap, **params)
    import ctypes
    from paper_2401_14762_b200 import _native
    lib = _native.load()
    ph = (ctypes.c_ulonglong * 16)()
    convex = args.algo in ("fista", "admm")
    dbg = lib.hcs_debug_phases_cx if convex else lib.hcs_debug_phases
    has_ph = dbg(ph, 1) == 0
    out = None
    for _ in range(args.reps):
        torch.cuda.synchronize()
        t = time.perf_counter()
        out = solve_batch(args.algo, y, m, b, cfg, out=out)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t
        it = out.iterations.cpu().numpy()
        print(f"{args.algo} k={args.kappa} P={cube.n_pixels}: {dt * 1e3:.2f} ms, {cube.n_pixels / dt:.0f} px/s, "
              f"iters mean {it.mean():.2f} max {it.max()} total {it.sum()}, {dt / max(it.sum(), 1) * 1e6:.2f} us/iter"
              + ("" if convex else f", spilled {int(out.workspace[16:24].view(torch.int64).item())}"))
        if has_ph:
            dbg(ph, 1)
            names = (["slots", "writeback", "gemm1", "epi1", "gemm2", "epi2"] if convex else
                     ["stop", "corr", "select", "gather", "gram", "chol", "solve", "post", "resid", "fallback",
                      "result", "diag0", "panel", "trail"])
            tot = sum(ph[:len(names)])
            print("  phases (% of CTA cycles): " + ", ".join(f"{nm} {100.0 * ph[i] / max(tot, 1):.1f}"
                                                           for i, nm in enumerate(names)))
            if convex and ph[7]:
                print(f"  sparse GEMM: {ph[6] / ph[7]:.3f} of the dense 4 x 8 blocks active, masked path on "
                      f"{ph[8] / max(ph[9], 1):.3f} of the ticks")
            nit = max(int(it.sum()), 1)
            print(f"  CTA cycles per pixel: {tot / cube.n_pixels:.0f} = " + ", ".join(
                f"{nm} {ph[i] / cube.n_pixels:.0f}" for i, nm in enumerate(names)))
            print(f"  CTA cycles per pixel-iteration: {tot / nit:.0f} = " + ", ".join(
                f"{nm} {ph[i] / nit:.0f}" for i, nm in enumerate(names)))
    if args.dump:
        np.savez(args.dump, x=out.x.cpu().numpy(), iterations=out.iterations.cpu().numpy(),
                 converged=out.converged.cpu().numpy(), failed_at=out.failed_at.cpu().numpy())


if __name__ == "__main__":
    main()
