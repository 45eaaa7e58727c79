"""Where does the end-to-end (host buffers) time of recover_cube go?  Profiling helper.

    python tools/e2e_probe.py [--algo fista --lam 100] [--reps 16]

Uses one 512x217 tile replicated `--reps` times along x (scaling-cube size at 16).
"""

import argparse
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2401_14762_b200 import synth  # noqa: E402
from paper_2401_14762_b200.solvers import SolverConfig, recover_cube, solve_batch  # noqa: E402
from paper_2401_14762_b200.transform import Dictionary  # noqa: E402


def tick(msg, t):
    torch.cuda.synchronize()
    now = time.perf_counter()
    print(f"  {msg:40s} {1e3 * (now - t):9.1f} ms", flush=True)
    return now


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--algo", default="fista")
    ap.add_argument("--lam", type=float, default=100.0)
    ap.add_argument("--kappa", type=int, default=27)
    ap.add_argument("--reps", type=int, default=16)
    ap.add_argument("--calls", type=int, default=3)
    args = ap.parse_args()
    tile = synth.generate(512, 217, 224, seed=0)
    y = np.concatenate([tile.y] * args.reps)
    masks = np.concatenate([tile.masks] * args.reps)
    P, m = y.shape
    X = 512 * args.reps
    params = dict(kappa=args.kappa) if args.algo in ("gomp", "biht", "cosamp") else dict(lam=args.lam)
    cfg = SolverConfig(time_limit=None, max_iter=2000, **params)
    y_h = torch.from_numpy(y.reshape(X, 217, m)).pin_memory()
    dic = Dictionary.per_pixel(tile.basis, masks)
    print(f"P={P}")
    for c in range(args.calls):
        dic._device = {}
        t = time.perf_counter()
        cube, st = recover_cube(y_h, dic, cfg, args.algo)
        tick(f"recover_cube call {c}", t)
    out = torch.empty((X, 217, 224), dtype=torch.float64, pin_memory=True)
    for c in range(args.calls):
        t = time.perf_counter()
        cube, st = recover_cube(y_h, dic, cfg, args.algo, out=out)
        tick(f"recover_cube(out=pinned) call {c}", t)
    for ch in (P, P // 4, P // 16):
        t = time.perf_counter()
        cube, st = recover_cube(y_h, dic, cfg, args.algo, out=out, chunk_pixels=ch)
        tick(f"recover_cube(out=pinned, chunk={ch})", t)
    # pieces
    t = time.perf_counter()
    host = torch.empty((P, 224), dtype=torch.float64, pin_memory=True)
    t = tick("pinned alloc x", t)
    host2 = torch.empty((P, 224), dtype=torch.float64, pin_memory=True)
    t = tick("pinned alloc x (2nd)", t)
    del host2
    yd = y_h.reshape(P, m).to("cuda", non_blocking=True)
    t = tick("H2D y (pinned)", t)
    md = torch.as_tensor(masks, device="cuda")
    t = tick("H2D masks (pageable)", t)
    bd = torch.as_tensor(tile.basis, device="cuda")
    b = solve_batch(args.algo, yd, md, bd, cfg)
    t = tick("solve_batch", t)
    host.copy_(b.x, non_blocking=True)
    t = tick("D2H x (pinned)", t)
    xn = b.x.cpu()
    t = tick("D2H x (pageable)", t)
    for name in ("iterations", "converged", "final_delta", "failed_at", "admm_gap", "elapsed"):
        getattr(b, name).cpu().numpy()
    t = tick("D2H stats (pageable)", t)


if __name__ == "__main__":
    main()
