"""Per-pixel iteration counts of one solver configuration on the scaling cube
(device-generated), saved for the slot-engine tail simulation (tools/tail_sim.py).

    python tools/iter_hist.py --algo admm --lam 0.1 --out gpurun_out/iters_admm.npy
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

ap = argparse.ArgumentParser()
ap.add_argument("--algo", default="admm")
ap.add_argument("--lam", type=float, default=0.1)
ap.add_argument("--kappa", type=int, default=27)
ap.add_argument("--cap", type=int, default=5000)
ap.add_argument("--out", required=True)
args = ap.parse_args()
dev = torch.device("cuda")
c = synth.generate_named_device("scaling", device=dev)
params = dict(lam=args.lam) if args.algo in ("fista", "admm") else dict(kappa=args.kappa)
cfg = SolverConfig(time_limit=None, max_iter=args.cap, **params)
b = solve_batch(args.algo, c.y, c.masks, torch.as_tensor(c.basis, device=dev), cfg)
torch.cuda.synchronize()
t = time.perf_counter()
b = solve_batch(args.algo, c.y, c.masks, torch.as_tensor(c.basis, device=dev), cfg, out=b)
torch.cuda.synchronize()
dt = time.perf_counter() - t
it = b.iterations.cpu().numpy()
np.save(args.out, it)
print(f"{args.algo} {params}: {dt * 1e3:.1f} ms, iterations total {it.sum()} mean {it.mean():.1f} "
      f"p99 {np.percentile(it, 99):.0f} p99.99 {np.percentile(it, 99.99):.0f} max {it.max()}")
