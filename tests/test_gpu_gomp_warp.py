"""The warp-per-pixel gOMP kernel (hcs_gomp_warp.cu) at its edges, against the
oracle (SURVEY.md §8(c) comparator: coefficients 1e-9, supports, iterations,
flags; tie exceptions replay-confirmed).

* every register-column instantiation (MR = 32, 48, 64, 80, 92, 96 rows) and
  M > 96 (the CTA kernel);
* kappa = 33 (one pre-column in every top system), kappa = 34 (CTA kernel),
  G = kappa (|S| > kappa from the second pass: pre-columns up to M);
* rank-deficient systems: an identity basis makes every column outside the
  pixel's mask a zero column of A, so the zero-fill refit is rank deficient and
  the reference falls back to gelsd's minimum-norm solution
  (kernels.py:61-66); the warp kernel's rank guard must hand those pixels to
  the CTA kernel's pivoted-QR / complete-orthogonal-decomposition path;
* non-finite and all-zero measurements, the time budget, and the iteration cap.
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import cpu_solvers as oc  # noqa: E402
from paper_2401_14762_b200 import synth  # noqa: E402
from paper_2401_14762_b200.solvers import SolverConfig, solve_batch  # noqa: E402
from parity import compare  # noqa: E402
from test_gpu_parity import decode_trace, make_replay  # noqa: E402

pytestmark = pytest.mark.gpu


def _cube(n, m, P, seed):
    """Synthetic spectra of n bands, each pixel measured at m random bands."""
    c = synth.generate(P // 10, 10, n, seed=seed)
    rng = np.random.default_rng(seed)
    masks = np.sort(np.argsort(rng.random((P, n)), axis=1)[:, :m], axis=1).astype(np.uint8)
    y = np.take_along_axis(c.spectra, masks.astype(np.intp), axis=1)
    return c.basis, np.ascontiguousarray(y), masks


def _check(basis, y, masks, kappa, G, cap=None, max_ties=0.02):
    dev = torch.device("cuda")
    cfg = SolverConfig(kappa=kappa, atoms_per_iter=G, time_limit=None, max_iter=cap)
    b = solve_batch("gomp", torch.as_tensor(y, device=dev), torch.as_tensor(masks, device=dev),
                    torch.as_tensor(basis, device=dev), cfg, trace_calls=64)
    torch.cuda.synchronize()
    got = dict(x=b.x.cpu().numpy(), iterations=b.iterations.cpu().numpy(),
               converged=b.converged.cpu().numpy().astype(bool), failed_at=b.failed_at.cpu().numpy(),
               trace=decode_trace((b.trace, b.trace_len), basis.shape[0]))
    ocfg = oc.OracleConfig(kappa=kappa, atoms_per_iter=G, max_iter=cap or 0)
    ref = oc.solve_cube("gomp", basis, y, masks, ocfg, jobs=8, trace=True)
    rep = compare(dict(x=ref.x, iterations=ref.iterations, converged=ref.converged, failed_at=ref.failed_at), got,
                  y, ref.traces, got["trace"], "gomp", replay=make_replay("gomp", basis, y, masks, ocfg))
    assert not rep["bad"], rep["bad"][:3]
    assert len(rep["ties"]) <= max(2, int(max_ties * len(y))), rep["ties"][:3]
    return b


@pytest.mark.parametrize("m", [24, 40, 60, 75, 90, 95, 120])
def test_every_register_column_size(m):
    n = 160 if m <= 90 else 224
    basis, y, masks = _cube(n, m, 240, seed=m)
    kappa = min(20, m - 2)
    _check(basis, y, masks, kappa, max(1, kappa // 5))


@pytest.mark.parametrize("kappa,G", [(33, 6), (34, 6), (12, 12), (30, 30)])
def test_pre_columns_and_the_cta_kernel(kappa, G):
    basis, y, masks = _cube(224, 90, 240, seed=kappa + G)
    _check(basis, y, masks, kappa, G, cap=8)


def test_rank_deficient_refits_take_the_minimum_norm_path():
    n, m, P = 48, 20, 160
    basis = np.eye(n)
    rng = np.random.default_rng(3)
    masks = np.sort(np.argsort(rng.random((P, n)), axis=1)[:, :m], axis=1).astype(np.uint8)
    x0 = np.zeros((P, n))
    for p in range(P):   # sparse coefficients on measured bands: A x0 = x0[mask]
        sel = rng.choice(masks[p], size=4, replace=False)
        x0[p, sel] = rng.uniform(0.5, 1.5, 4) * rng.choice([-1, 1], 4)
    y = np.ascontiguousarray(np.take_along_axis(x0, masks.astype(np.intp), axis=1))
    b = _check(basis, y, masks, kappa=8, G=2, cap=6)
    assert int(b.workspace[16:24].view(torch.int64).item()) > 0   # pixels went to the CTA kernel


def test_flags_budget_and_cap():
    basis, y, masks = _cube(224, 90, 60, seed=5)
    y = y.copy()
    y[3] = 0.0                  # y = 0 shortcut: converged, 0 iterations
    dev = torch.device("cuda")
    cfg = SolverConfig(kappa=27, atoms_per_iter=5, time_limit=None, max_iter=1)
    b = solve_batch("gomp", torch.as_tensor(y, device=dev), torch.as_tensor(masks, device=dev),
                    torch.as_tensor(basis, device=dev), cfg)
    it = b.iterations.cpu().numpy()
    assert it[3] == 0 and bool(b.converged[3].item())
    assert np.all(np.delete(it, 3) == 1) and not b.converged.cpu().numpy()[np.arange(60) != 3].any()
    # an expired budget: every pixel stops before its first pass (timeout, not converged)
    cfg = SolverConfig(kappa=27, atoms_per_iter=5, time_limit=1e-9, max_iter=100)
    b = solve_batch("gomp", torch.as_tensor(y, device=dev), torch.as_tensor(masks, device=dev),
                    torch.as_tensor(basis, device=dev), cfg)
    it = b.iterations.cpu().numpy()
    assert np.all(np.delete(it, 3) == 0) and not b.converged.cpu().numpy()[np.arange(60) != 3].any()
    # non-finite measurements: ValueError, as scipy's finiteness check in the reference
    y[7, 2] = np.nan
    with pytest.raises(ValueError):
        solve_batch("gomp", torch.as_tensor(y, device=dev), torch.as_tensor(masks, device=dev),
                    torch.as_tensor(basis, device=dev), SolverConfig(kappa=27, time_limit=None))
