"""Whole-cube parity at BASELINE.json's full config sizes.

Every pixel of the cfg1 / cfg2 cube (Jasper-shaped, 100 x 100 x 198) and of
the cfg3 cube (China-shaped, 420 x 140 x 154) goes through the GPU path and
through the CPU oracle (all host cores).  Pixels that disagree in coefficients,
iterations or flags are classified with selection traces from both sides: each
must be a roundoff-degenerate tie on the oracle side AND be reproduced by the
forced-selection replay; anything else is a real mismatch and fails the test.
The cube PSNR over the agreeing pixels must match to 0.01 dB, and for solvers
without tie exceptions the whole-cube PSNR must too.

gOMP's whole-cube PSNR is not roundoff-stable even for the oracle itself: its
second pass selects atoms from A^T r with r at roundoff level, and the tie
pixels carry most of the squared error.  For gOMP the whole cube is therefore
judged against the oracle's own roundoff band: an ensemble of oracle re-solves
of y (1 + 2^-52 N(0,1)) (tools/cube_parity.py --ensemble,
profiles/gomp_ls_statistics_r02.txt).  The GPU must not disagree with the
oracle on more pixels than 1.3 x the ensemble's largest flip count (the
round-1 normal-equations solver failed this at 2.5x: a systematic bias, not
roundoff), and its cube dPSNR must lie inside the ensemble's range (with the
oracle itself, dPSNR 0) widened by 25% of its width on each side -- with n
exchangeable draws a further draw falls outside their range with probability
2 / (n + 1), which the widening absorbs.
"""

import math
import multiprocessing
import os
from concurrent.futures import ProcessPoolExecutor

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import cpu_solvers as oc  # noqa: E402
from paper_2401_14762_b200 import synth  # noqa: E402
from paper_2401_14762_b200.solvers import SolverConfig, solve_batch  # noqa: E402
from parity import compare  # noqa: E402
from test_gpu_parity import decode_trace, make_replay  # noqa: E402

pytestmark = pytest.mark.gpu

ENSEMBLE = 6

CASES = [
    ("jasper", "gomp", dict(kappa=24, atoms_per_iter=4), None, 0.02),       # cfg1
    ("jasper", "fista", dict(lam=100.0), 5000, 0.0),                        # cfg2
    ("jasper", "admm", dict(lam=100.0, alpha=1.8), 5000, 0.0),              # cfg2
    ("jasper", "fista", dict(lam=0.1), 5000, 0.0),                          # cfg2 / cfg5 lambda
    ("china", "biht", dict(kappa=22, mu=0.1), 2000, 0.0),                   # cfg3
    ("china", "gomp", dict(kappa=22, atoms_per_iter=4), None, 0.02),        # cfg3
]


@pytest.fixture(scope="module")
def pool():
    cores = max(1, len(os.sched_getaffinity(0)))
    # forkserver: the workers must not inherit this process's CUDA context
    ctx = multiprocessing.get_context("forkserver")
    with ProcessPoolExecutor(max_workers=cores, initializer=oc.single_thread_blas, mp_context=ctx) as p:
        yield p, cores


@pytest.fixture(scope="module")
def cubes():
    return {}


def _db(sse, peak, count):
    mse = sse / count
    return math.inf if mse == 0 else 10.0 * math.log10(peak * peak / mse)


@pytest.mark.parametrize("cube_name,algo,params,cap,max_tie_frac", CASES)
def test_full_cube_parity(pool, cubes, cube_name, algo, params, cap, max_tie_frac):
    ex, cores = pool
    if cube_name not in cubes:
        cubes[cube_name] = synth.generate_named(cube_name, workers=min(16, cores))
    c = cubes[cube_name]
    dev = torch.device("cuda")
    cfg = SolverConfig(time_limit=None, max_iter=cap, **params)
    basis_d = torch.as_tensor(c.basis, device=dev)
    b = solve_batch(algo, torch.as_tensor(c.y, device=dev), torch.as_tensor(c.masks, device=dev), basis_d, cfg)
    torch.cuda.synchronize()
    gx, git = b.x.cpu().numpy(), b.iterations.cpu().numpy()
    gconv, gfail = b.converged.cpu().numpy().astype(bool), b.failed_at.cpu().numpy()
    ocfg = oc.OracleConfig(max_iter=cap or 0, **params)
    ref = oc.solve_cube(algo, c.basis, c.y, c.masks, ocfg, pool=ex, chunk=256)
    nr = np.linalg.norm(ref.x, axis=1)
    err = np.linalg.norm(gx - ref.x, axis=1)
    coef_bad = np.where(nr > 0, err > 1e-9 * nr, err > 1e-12)
    bad = coef_bad | (git != ref.iterations) | (gconv != ref.converged) | (gfail != ref.failed_at)
    idx = np.flatnonzero(bad)
    assert len(idx) <= max_tie_frac * c.n_pixels, f"{len(idx)} disagreeing pixels"
    if len(idx):
        # classify every disagreeing pixel: traces from both sides + forced-selection replay
        y, m = np.ascontiguousarray(c.y[idx]), np.ascontiguousarray(c.masks[idx])
        bt = solve_batch(algo, torch.as_tensor(y, device=dev), torch.as_tensor(m, device=dev), basis_d, cfg,
                         trace_calls=64)
        torch.cuda.synchronize()
        got = dict(x=bt.x.cpu().numpy(), iterations=bt.iterations.cpu().numpy(),
                   converged=bt.converged.cpu().numpy().astype(bool), failed_at=bt.failed_at.cpu().numpy(),
                   trace=decode_trace((bt.trace, bt.trace_len), c.n))
        rt = oc.solve_cube(algo, c.basis, y, m, ocfg, pool=ex, trace=True, chunk=16)
        rep = compare(dict(x=rt.x, iterations=rt.iterations, converged=rt.converged, failed_at=rt.failed_at), got,
                      y, rt.traces, got["trace"], algo, replay=make_replay(algo, c.basis, y, m, ocfg))
        assert not rep["bad"], rep["bad"][:3]
        assert all(t.get("replay_ok") for t in rep["ties"])
    # PSNR: the agreeing pixels exactly; the whole cube when nothing disagrees
    rec_g, rec_r = gx @ c.basis.T, ref.x @ c.basis.T
    sse_g = np.einsum("pn,pn->p", c.spectra - rec_g, c.spectra - rec_g)
    sse_r = np.einsum("pn,pn->p", c.spectra - rec_r, c.spectra - rec_r)
    peak = float(np.max(np.abs(c.spectra)))
    ok = ~bad
    pg, pr = _db(sse_g[ok].sum(), peak, ok.sum() * c.n), _db(sse_r[ok].sum(), peak, ok.sum() * c.n)
    assert abs(pg - pr) <= 0.01 or (pg > 200 and pr > 200), (pg, pr)
    if not len(idx):
        assert abs(_db(sse_g.sum(), peak, c.spectra.size) - _db(sse_r.sum(), peak, c.spectra.size)) <= 0.01
    if algo == "gomp":
        p_ref = _db(sse_r.sum(), peak, c.spectra.size)
        dps, flips = [0.0], []
        for e in range(ENSEMBLE):
            rng = np.random.default_rng(100 + e)
            yp = c.y * (1.0 + 2.0 ** -52 * rng.standard_normal(c.y.shape))
            rp = oc.solve_cube(algo, c.basis, yp, c.masks, ocfg, pool=ex, chunk=256)
            d_p = c.spectra - rp.x @ c.basis.T
            dps.append(_db(float(np.einsum("pn,pn->", d_p, d_p)), peak, c.spectra.size) - p_ref)
            flips.append(int((rp.iterations != ref.iterations).sum()))
        dp_gpu = _db(sse_g.sum(), peak, c.spectra.size) - p_ref
        lo, hi = min(dps), max(dps)
        print(f"  gOMP band: GPU dPSNR {dp_gpu:+.2f} dB, {len(idx)} disagreeing; oracle ensemble dPSNR "
              f"[{lo:+.2f}, {hi:+.2f}] dB, flips {flips}")
        assert len(idx) <= 1.3 * max(flips), (len(idx), flips)
        assert lo - 0.25 * (hi - lo) <= dp_gpu <= hi + 0.25 * (hi - lo), (dp_gpu, dps)
    print(f"{cube_name} {algo} {params}: {c.n_pixels} px, {len(idx)} replay-confirmed tie exceptions, "
          f"agreeing-pixel PSNR {pg:.4f} / {pr:.4f} dB")
