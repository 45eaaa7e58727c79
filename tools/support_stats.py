"""Support statistics of converged FISTA/ADMM iterates (diagnostics for
k-step skipping in the slot engine): per group of 32 pixels, the fraction of
the N_pad/4 DMMA k-steps whose 4 coefficient rows are nonzero in any pixel."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2401_14762_b200 import synth  # noqa: E402
from paper_2401_14762_b200.solvers import SolverConfig, solve_batch  # noqa: E402

c = synth.generate_named_device("salinas", device="cuda")
for algo, lam in (("fista", 0.1), ("admm", 0.1)):
    b = solve_batch(algo, c.y, c.masks, torch.as_tensor(c.basis, device="cuda"),
                    SolverConfig(lam=lam, time_limit=None, max_iter=5000))
    x = b.x.cpu().numpy()
    nz = x != 0
    per_px = nz.sum(axis=1)
    P, n = x.shape
    ks = (n + 15) // 16 * 4
    g = nz[: P // 32 * 32].reshape(-1, 32, n).any(axis=1)           # union over 32 pixels
    g = np.pad(g, ((0, 0), (0, ks * 4 - n))).reshape(g.shape[0], ks, 4).any(axis=2)
    print(f"{algo} lam={lam}: nonzeros per pixel mean {per_px.mean():.1f} p90 {np.percentile(per_px, 90):.0f} "
          f"max {per_px.max()}; active k-steps per 32-pixel group mean {g.mean():.3f} (of {ks}); "
          f"coefficient-index histogram (nonzero share per 16-band bin): "
          + " ".join(f"{v:.2f}" for v in nz.mean(axis=0).reshape(-1, 16).mean(axis=1)))
