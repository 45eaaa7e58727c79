"""GPU vs oracle parity report on a synthetic cube slice (diagnostics)."""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import cpu_solvers as oc  # noqa: E402
from paper_2401_14762_b200 import synth  # noqa: E402
from paper_2401_14762_b200.solvers import SolverConfig, solve_batch  # noqa: E402
from parity import compare  # noqa: E402
from test_gpu_parity import decode_trace, make_replay  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--cube", default="salinas")
ap.add_argument("--algo", default="gomp")
ap.add_argument("--kappa", type=int, default=27)
ap.add_argument("--lam", type=float, default=0.1)
ap.add_argument("--cap", type=int, default=2000)
ap.add_argument("--pixels", type=int, default=3000)
args = ap.parse_args()
n = synth.CUBES[args.cube]["n"]
c = synth.generate(args.pixels // 50, 50, n, seed=99)
greedy = args.algo in ("gomp", "biht", "cosamp")
params = dict(kappa=args.kappa) if greedy else dict(lam=args.lam)
cfg = SolverConfig(time_limit=None, max_iter=args.cap if args.algo != "gomp" else None, **params)
dev = torch.device("cuda")
b = solve_batch(args.algo, torch.as_tensor(c.y, device=dev), torch.as_tensor(c.masks, device=dev),
                torch.as_tensor(c.basis, device=dev), cfg, trace_calls=64 if greedy else 0)
got = dict(x=b.x.cpu().numpy(), iterations=b.iterations.cpu().numpy(), converged=b.converged.cpu().numpy().astype(bool),
           failed_at=b.failed_at.cpu().numpy())
if greedy:
    got["trace"] = decode_trace((b.trace, b.trace_len), n)
ref = oc.solve_cube(args.algo, c.basis, c.y, c.masks, oc.OracleConfig(max_iter=cfg.max_iter or 0, **params),
                    jobs=16, trace=greedy)
ocfg = oc.OracleConfig(max_iter=cfg.max_iter or 0, **params)
rep = compare(dict(x=ref.x, iterations=ref.iterations, converged=ref.converged, failed_at=ref.failed_at), got, c.y,
              ref.traces, got.get("trace"), args.algo, replay=make_replay(args.algo, c.basis, c.y, c.masks, ocfg))
it_diff = int((ref.iterations != got["iterations"]).sum())
print(json.dumps({"algo": args.algo, "kappa": args.kappa, "pixels": c.n_pixels, "bad": len(rep["bad"]),
                  "ties": len(rep["ties"]), "ties_replay_ok": sum(1 for t in rep["ties"] if t.get("replay_ok")), "iteration_mismatches": it_diff, "worst_rel": rep["worst_rel"],
                  "iters_gpu": int(got["iterations"].sum()), "iters_oracle": int(ref.iterations.sum()),
                  "bad_examples": rep["bad"][:3], "tie_examples": rep["ties"][:3]}, default=str))
