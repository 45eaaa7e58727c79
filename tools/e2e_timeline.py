"""Where do the host-side milliseconds of one recover_cube call go?  Wall-clock
marks around the phases of the host pipeline (diagnostics).

    python tools/e2e_timeline.py [--algo gomp --kappa 27]
"""
import argparse
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

from paper_2401_14762_b200 import solvers, synth  # noqa: E402
from paper_2401_14762_b200.solvers import SolverConfig, recover_cube, solve_batch  # noqa: E402
from paper_2401_14762_b200.transform import Dictionary  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--algo", default="gomp")
ap.add_argument("--kappa", type=int, default=27)
ap.add_argument("--lam", type=float, default=0.1)
args = ap.parse_args()
dev = torch.device("cuda")
c = synth.generate_named_device("scaling", device=dev)
X, Y = c.shape
n, m = c.n, c.m
y_h = torch.from_numpy(c.y.cpu().numpy().reshape(X, Y, m)).pin_memory()
dic = Dictionary.per_pixel(c.basis, c.masks.cpu().numpy())
out = torch.empty((X, Y, n), dtype=torch.float64, pin_memory=True)
params = dict(lam=args.lam) if args.algo in ("fista", "admm") else dict(kappa=args.kappa)
cfg = SolverConfig(time_limit=None, max_iter=2000, **params)

marks = []
orig_host, orig_stats = solvers._recover_host, solvers._stats_from_batch


def host(*a, **k):
    t = time.perf_counter()
    r = orig_host(*a, **k)
    marks.append(("_recover_host returned (device work enqueued, host waited for streams)", time.perf_counter() - t))
    t = time.perf_counter()
    torch.cuda.synchronize()
    marks.append(("sync after _recover_host", time.perf_counter() - t))
    return r


def stats(*a, **k):
    t = time.perf_counter()
    r = orig_stats(*a, **k)
    marks.append(("_stats_from_batch (per-pixel stats D2H + aggregates)", time.perf_counter() - t))
    return r


solvers._recover_host, solvers._stats_from_batch = host, stats
for rep in range(3):
    marks.clear()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    recover_cube(y_h, dic, cfg, args.algo, out=out)
    torch.cuda.synchronize()
    total = time.perf_counter() - t0
    b = solve_batch(args.algo, c.y, c.masks, torch.as_tensor(c.basis, device=dev), cfg)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    solve_batch(args.algo, c.y, c.masks, torch.as_tensor(c.basis, device=dev), cfg, out=b)
    torch.cuda.synchronize()
    dev_t = time.perf_counter() - t1
    print(f"rep {rep}: recover_cube {1e3 * total:.1f} ms, device-only solve_batch {1e3 * dev_t:.1f} ms")
    for k, v in marks:
        print(f"   {1e3 * v:8.1f} ms  {k}")
