"""Small cases of every kernel family, for compute-sanitizer.

    compute-sanitizer --tool memcheck  python tools/sanitize_cases.py
    compute-sanitizer --tool racecheck python tools/sanitize_cases.py
    compute-sanitizer --tool synccheck python tools/sanitize_cases.py

Covers: the convex slot engines (FISTA / ADMM, 32 slots and the 16-slot
engine of high sampling ratios), the certified zero-shrinkage ADMM pass, the
greedy CTA kernel for gOMP / BIHT / CoSaMP (shared-memory systems and, with
HCS_GREEDY_CAP_KB=16, systems spilled to the global scratch), the
warp-per-pixel gOMP kernel with its spill list, the mask validation (a bad
mask), the input side (synth spectra, sparsify + measure), the PSNR kernels,
the batched kernels and the basis check.  Exits 0 when every case ran.
"""

import ctypes
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2401_14762_b200 import _native as nat  # noqa: E402
from paper_2401_14762_b200 import kernels as gk  # noqa: E402
from paper_2401_14762_b200 import metrics, sparsify, synth  # noqa: E402
from paper_2401_14762_b200.solvers import SolverConfig, solve_batch  # noqa: E402


def run(algo, c, cfg, masks=None, expect_error=False):
    dev = torch.device("cuda")
    m = c.masks if masks is None else masks
    try:
        b = solve_batch(algo, torch.as_tensor(c.y, device=dev), torch.as_tensor(m, device=dev),
                        torch.as_tensor(c.basis, device=dev), cfg)
        torch.cuda.synchronize()
        assert not expect_error, "bad mask accepted"
        return b
    except ValueError:
        if not expect_error:
            raise
        return None


def main():
    lib = nat.load()
    dev = torch.device("cuda")
    c224 = synth.generate(6, 8, 224, seed=3)          # 48 px, N = 224, M = 90
    c154 = synth.generate(5, 8, 154, seed=4)          # 40 px, N = 154, M = 62
    cases = [
        ("fista", c224, SolverConfig(lam=0.1, time_limit=None, max_iter=300)),
        ("admm", c224, SolverConfig(lam=0.1, time_limit=None, max_iter=300)),
        ("admm", c224, SolverConfig(lam=100.0, time_limit=None, max_iter=300)),   # zero-shrinkage pass
        ("fista", c154, SolverConfig(lam=100.0, time_limit=None, max_iter=300)),
        ("gomp", c224, SolverConfig(kappa=27, atoms_per_iter=5, time_limit=None)),   # warp kernel + spills
        ("gomp", c224, SolverConfig(kappa=33, atoms_per_iter=6, time_limit=None)),
        ("gomp", c154, SolverConfig(kappa=22, atoms_per_iter=4, time_limit=None)),
        ("gomp", c224, SolverConfig(kappa=12, atoms_per_iter=12, time_limit=None, max_iter=6)),   # pre-columns, spills
        ("biht", c224, SolverConfig(kappa=27, time_limit=None, max_iter=200)),
        ("biht", c224, SolverConfig(kappa=33, time_limit=None, max_iter=200)),
        ("cosamp", c224, SolverConfig(kappa=27, time_limit=None, max_iter=200)),
        ("cosamp", c224, SolverConfig(kappa=33, time_limit=None, max_iter=200)),
    ]
    for algo, c, cfg in cases:
        run(algo, c, cfg)
        print(f"ok {algo} N={c.n} {cfg.lam if algo in ('fista', 'admm') else cfg.kappa}", flush=True)
    # greedy systems in the global scratch (shared LS region trimmed to 16 KB)
    os.environ["HCS_GREEDY_CAP_KB"] = "16"
    for algo in ("biht", "cosamp"):
        run(algo, c224, SolverConfig(kappa=27, time_limit=None, max_iter=100))
    os.environ["HCS_GOMP_WARP"] = "0"
    run("gomp", c224, SolverConfig(kappa=27, atoms_per_iter=5, time_limit=None))   # CTA pivoted-QR path
    del os.environ["HCS_GREEDY_CAP_KB"], os.environ["HCS_GOMP_WARP"]
    print("ok global-scratch greedy + CTA gOMP", flush=True)
    # the 16-slot convex engine (N = 224, M = 224: 32 slots exceed shared memory)
    rng = np.random.default_rng(1)
    full = synth.SyntheticCube(basis=c224.basis, coeffs=c224.coeffs, spectra=c224.spectra,
                               masks=np.tile(np.arange(224, dtype=np.uint8), (48, 1)), y=c224.spectra.copy(),
                               shape=(48, 1), seeds=c224.seeds)
    run("fista", full, SolverConfig(lam=0.1, time_limit=None, max_iter=100))
    run("admm", full, SolverConfig(lam=0.1, time_limit=None, max_iter=100))
    print("ok 16-slot engines", flush=True)
    # invalid masks: validated, every solver kernel exits
    bad = c224.masks.copy()
    bad[3, 4] = bad[3, 3]
    for algo in ("fista", "admm", "gomp", "biht", "cosamp"):
        run(algo, c224, SolverConfig(kappa=20, time_limit=None, max_iter=10), masks=bad, expect_error=True)
    print("ok mask validation", flush=True)
    # input side + PSNR + batched kernels + basis check
    inp = synth.generate_device(8, 8, 224, seed=5, with_coeffs=True, device=dev)
    sse = torch.zeros(1, dtype=torch.float64, device=dev)
    metrics.sse_coeff_partials(inp.coeffs, inp.coeffs * 0.5, out=sse)
    basis_d = torch.as_tensor(inp.basis, device=dev)
    metrics.psnr_partials(inp.spectra, inp.coeffs, basis_d)
    sparsify.sparsify_measure(inp.spectra, basis_d, 90, rule="meanstd", factor=0.5,
                              keys=torch.rand((64, 224), dtype=torch.float64, device=dev))
    gk.soft_threshold(rng.standard_normal(1000), 0.3)
    gk.argmax_k(rng.standard_normal((7, 224)), 33)
    gk.least_squares(rng.standard_normal((5, 90, 40)), rng.standard_normal((5, 90)))
    gk.least_squares(rng.standard_normal((3, 200, 180)), rng.standard_normal((3, 200)))   # global scratch
    gk.residual_delta(rng.standard_normal((4, 90)), rng.standard_normal((4, 90)))
    gk.lipschitz_batch(c224.basis, c224.masks[:8])
    out = ctypes.c_double()
    assert lib.hcs_check_basis(224, basis_d.data_ptr(), ctypes.byref(out), None) == 0
    torch.cuda.synchronize()
    print("ok input side / psnr / batched kernels", flush=True)


if __name__ == "__main__":
    main()
