"""Generate the golden fixtures in this directory FROM THE REFERENCE ITSELF.

Run in the build container (the reference is importable there, not on the GPU
box):  python tests/golden/make_golden.py

For every case it builds seeded synthetic inputs (paper_2401_14762_b200.synth,
generator v1), picks a spread of pixels, and calls the unmodified reference
solver per pixel exactly as SURVEY.md §8(c) prescribes:

    SOLVERS[algo](y_p, Dictionary.from_matrix(Psi[mask_p]), SolverConfig(..., time_limit=None))

(`/root/reference/pkg/src/hypercs/solvers.py:397-403`, `transform.py:245-251`).
The reference computes in complex128; the fixtures keep x.real (x.imag is
checked to be exactly zero).  Kernel-level fixtures come from
`hypercs.kernels` (`kernels.py:14-76`) and `lipschitz_constant`
(`transform.py:176-217`).

The fixtures pin the CPU oracle (`oracle/cpu_solvers.py`) and the GPU path.
Inputs are stored verbatim (y, masks) so nothing depends on regenerating them;
the basis is rebuilt by `synth.dct_basis` (libm cosines, bit-stable).
"""

import json
import math
import os
import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, "/root/reference/pkg/src")

import hypercs  # noqa: E402  (the reference package, read-only)
from hypercs import Dictionary, SolverConfig, SOLVERS  # noqa: E402
from hypercs import kernels as ref_kernels  # noqa: E402
from hypercs.transform import lipschitz_constant  # noqa: E402
import hypercs.solvers as ref_solvers  # noqa: E402

_TRACE = []
_argmax_k = ref_solvers.argmax_k


def _traced_argmax_k(v, k):
    """Records every selection the reference solvers make (the survey's
    instrumentation): (k, picked, max|v|, k-th gap)."""
    picked = _argmax_k(v, k)
    mag = np.sort(np.abs(np.asarray(v)))[::-1]
    gap = float(mag[k - 1] - mag[k]) if k < mag.size else math.inf
    _TRACE.append([int(k), [int(i) for i in picked], float(mag[0]), gap])
    return picked


ref_solvers.argmax_k = _traced_argmax_k

from paper_2401_14762_b200 import synth  # noqa: E402

PIXELS = 48

# name -> (cube, algo, params, cap)
CASES = {
    "cfg1_gomp_k24": ("jasper", "gomp", dict(kappa=24, atoms_per_iter=4), None),
    "cfg2_fista_l100": ("jasper", "fista", dict(lam=100.0), 5000),
    "cfg2_admm_l100": ("jasper", "admm", dict(lam=100.0, alpha=1.8), 5000),
    "cfg2_fista_l0.1": ("jasper", "fista", dict(lam=0.1), 5000),
    "cfg2_admm_l0.1": ("jasper", "admm", dict(lam=0.1, alpha=1.8), 5000),
    "cfg3_biht_k22": ("china", "biht", dict(kappa=22, mu=0.1), 2000),
    "cfg3_gomp_k22": ("china", "gomp", dict(kappa=22, atoms_per_iter=4), None),
    "cfg4_cosamp_k33": ("salinas", "cosamp", dict(kappa=33), 2000),
    "cfg5_cosamp_k27": ("salinas", "cosamp", dict(kappa=27), 2000),
    "cfg5_gomp_k27": ("salinas", "gomp", dict(kappa=27, atoms_per_iter=5), None),
    "cfg5_gomp_k33": ("salinas", "gomp", dict(kappa=33, atoms_per_iter=6), None),
    "cfg5_biht_k27": ("salinas", "biht", dict(kappa=27, mu=0.1), 2000),
    "cfg5_biht_k33": ("salinas", "biht", dict(kappa=33, mu=0.1), 2000),
}


def _small_cube(name, seed):
    """A small tile with the named cube's band count (same generator)."""
    n = synth.CUBES[name]["n"]
    return synth.generate(24, 24, n, seed=seed)


def solve_case(name, cube_name, algo, params, cap):
    cube = _small_cube(cube_name, seed=1000 + list(CASES).index(name))
    P = cube.n_pixels
    pick = np.linspace(0, P - 1, PIXELS).astype(np.int64)
    y = cube.y[pick].copy()
    masks = cube.masks[pick].copy()
    # edge cases folded into every case: an all-zero pixel, and (fista) a NaN
    # pixel that must fail at iteration 1 (`test_solvers.py:224-229`).  ADMM
    # cannot take one: its cho_solve raises ValueError on non-finite input
    # (`solvers.py:227`), which aborts the whole cube; recorded below.
    y[3] = 0.0
    if algo == "fista":
        y[5, 0] = np.nan
    basis = cube.basis
    cfg = SolverConfig(time_limit=None, max_iter=cap, **params)
    xs, its, conv, delta, gap, failed, lips, traces = [], [], [], [], [], [], [], []
    t0 = time.perf_counter()
    for p in range(PIXELS):
        d = Dictionary.from_matrix(basis[masks[p].astype(np.intp), :])
        lips.append(d.lipschitz)
        _TRACE.clear()
        try:
            r = SOLVERS[algo](y[p], d, cfg)
        except hypercs.NumericalFailure as exc:
            traces.append(list(_TRACE))
            xs.append(np.zeros(cube.n))
            its.append(0), conv.append(False), delta.append(math.nan), gap.append(math.nan)
            failed.append(exc.iteration)
            continue
        traces.append(list(_TRACE))
        assert not np.any(r.x.imag), "reference returned a non-real x"
        xs.append(r.x.real.copy())
        its.append(r.iterations)
        conv.append(r.converged)
        delta.append(r.final_delta)
        gap.append(math.nan if r.admm_gap is None else r.admm_gap)
        failed.append(-1)
    elapsed = time.perf_counter() - t0
    nan_error = ""
    if algo == "admm":
        bad = y[0].copy()
        bad[0] = np.nan
        try:
            SOLVERS[algo](bad, Dictionary.from_matrix(basis[masks[0].astype(np.intp), :]), cfg)
        except hypercs.NumericalFailure:
            nan_error = "NumericalFailure"
        except ValueError:
            nan_error = "ValueError"
    meta = dict(nan_error=nan_error, case=name, cube=cube_name, algo=algo, params=params, max_iter=cap,
                generator=synth.GENERATOR_VERSION, seed=int(cube.seeds[0]), tile=[24, 24],
                pixels=pick.tolist(), reference_elapsed_s=elapsed,
                numpy=np.__version__, python=sys.version.split()[0])
    np.savez_compressed(
        HERE / f"{name}.npz",
        n=np.int64(cube.n), y=y, masks=masks, x=np.array(xs), iterations=np.array(its, np.int32),
        converged=np.array(conv), final_delta=np.array(delta), admm_gap=np.array(gap),
        failed_at=np.array(failed, np.int32), lipschitz=np.array(lips),
        meta=np.array(json.dumps(meta)), traces=np.array(json.dumps(traces)),
    )
    print(f"{name}: {PIXELS} px in {elapsed:.1f}s, iters mean {np.mean(its):.1f} max {max(its)}")


def kernel_fixtures():
    """Known-answer vectors from hypercs.kernels on seeded real inputs."""
    rng = np.random.default_rng(77)
    out = {}
    # soft threshold (kernels.py:14-28)
    v = np.concatenate([rng.standard_normal(61) * 3.0, [0.0, 1.0, -1.0, 0.5, -0.5]])
    for i, t in enumerate((0.0, 0.5, 1.0, 2.5)):
        out[f"soft_v"] = v
        out[f"soft_t{i}"] = np.float64(t)
        out[f"soft_out{i}"] = ref_kernels.soft_threshold(v, t)
    # top-k with ties (kernels.py:31-41)
    ties = np.round(rng.standard_normal(200) * 4.0) / 4.0   # many exact ties
    out["argk_v"] = ties
    for k in (1, 4, 22, 66, 200):
        out[f"argk_out{k}"] = ref_kernels.argmax_k(ties, k)
    # least squares (kernels.py:44-67): full-rank, square, duplicate column,
    # zero column, underdetermined; real matrices
    cases = []
    for (m, k) in ((79, 24), (90, 66), (62, 22), (40, 40), (30, 5)):
        cases.append(rng.standard_normal((m, k)))
    col = rng.standard_normal(20)
    cases.append(np.stack([col, col, rng.standard_normal(20)], axis=1))   # duplicate
    zc = rng.standard_normal((25, 6))
    zc[:, 2] = 0.0
    cases.append(zc)                                                       # zero column
    cases.append(rng.standard_normal((7, 12)))                             # underdetermined
    for i, b in enumerate(cases):
        y = rng.standard_normal(b.shape[0])
        out[f"ls_b{i}"] = b
        out[f"ls_y{i}"] = y
        out[f"ls_s{i}"] = ref_kernels.least_squares(b, y).real
    out["ls_count"] = np.int64(len(cases))
    # Lipschitz constants of masked DCT bases (transform.py:176-217)
    lips = []
    for n in (154, 198, 224):
        basis = synth.dct_basis(n)
        for seed in range(4):
            mask = np.sort(np.random.default_rng(seed).choice(n, synth.measured_count(n), replace=False))
            lips.append((n, seed, lipschitz_constant(basis[mask, :].astype(np.complex128))))
    out["lip_table"] = np.array(lips)
    np.savez_compressed(HERE / "kernels.npz", **out)
    print("kernels.npz written")


def main():
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    kernel_fixtures()
    only = sys.argv[1:]
    for name, (cube_name, algo, params, cap) in CASES.items():
        if only and name not in only:
            continue
        solve_case(name, cube_name, algo, params, cap)


if __name__ == "__main__":
    main()
