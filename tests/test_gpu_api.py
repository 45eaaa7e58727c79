"""Reference behaviour through the public API on the GPU.

Each test restates a hypercs test (`/root/reference/pkg/tests/test_solvers.py`,
`test_kernels.py`, `test_acceptance.py`) with a real orthonormal dictionary
(the reference's tests use complex DFT dictionaries, which the real-FP64
device path does not take)."""

import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import paper_2401_14762_b200 as hcs  # noqa: E402
from oracle import cpu_solvers as oc  # noqa: E402
from paper_2401_14762_b200 import synth  # noqa: E402
from paper_2401_14762_b200.transform import Dictionary  # noqa: E402

pytestmark = pytest.mark.gpu
NO_LIMITS = dict(time_limit=None, max_iter=2000)


def partial_dct(n, m, seed):
    """Seeded selection of m of n orthonormal DCT-II rows (helpers.py:13-18, real basis)."""
    mask = hcs.build_selection_mask(n, m / n, seed)
    assert mask.m == m
    return hcs.build_dictionary(hcs.build_dct_basis(n), mask)


def planted(n, m, kappa, seed):
    rng = np.random.default_rng(seed)
    d = partial_dct(n, m, seed)
    x0 = np.zeros(n)
    x0[rng.choice(n, size=kappa, replace=False)] = rng.uniform(1.0, 2.0, size=kappa) * rng.choice([-1, 1], kappa)
    return d, x0, d.matrix @ x0


def test_identity_dictionary_closed_form():            # test_solvers.py:105-114, C4
    d = Dictionary.from_matrix(np.eye(3))
    y = np.array([2.0, 0.1, -3.0])
    for solver in (hcs.fista, hcs.admm):
        r = solver(y, d, hcs.SolverConfig(lam=0.5, epsilon=1e-10, time_limit=None, max_iter=50000))
        assert r.converged
        np.testing.assert_allclose(r.x, [1.5, 0.0, -2.5], atol=1e-6)


def test_fista_and_admm_reach_the_same_objective():     # test_solvers.py:116-122, C1
    for seed in range(5):
        d, _, y = planted(24, 10, 4, seed)
        for lam in (0.1, 100.0):
            cfg = hcs.SolverConfig(lam=lam, time_limit=None, max_iter=200000)
            h_f = hcs.lasso_objective(hcs.fista(y, d, cfg).x, y, d, lam)
            h_a = hcs.lasso_objective(hcs.admm(y, d, cfg).x, y, d, lam)
            assert abs(h_f - h_a) <= 1e-6 * max(1.0, abs(h_f))


def test_admm_reports_the_primal_gap():                 # test_solvers.py:132-136
    d, _, y = planted(16, 7, 3, 1)
    r = hcs.admm(y, d, hcs.SolverConfig(lam=0.1, **NO_LIMITS))
    assert r.admm_gap is not None and r.admm_gap >= 0.0
    assert hcs.fista(y, d, hcs.SolverConfig(lam=0.1, **NO_LIMITS)).admm_gap is None


@pytest.mark.parametrize("name", ["fista", "admm", "gomp", "biht", "cosamp"])
def test_zero_measurements_short_circuit(name):         # test_solvers.py:138-144, 161-165
    d = partial_dct(16, 7, 0)
    r = hcs.SOLVERS[name](np.zeros(7), d, hcs.SolverConfig(kappa=2))
    assert r.converged and r.iterations == 0 and r.final_delta == 0.0
    np.testing.assert_array_equal(r.x, np.zeros(16))


@pytest.mark.parametrize("name", ["gomp", "biht", "cosamp"])
def test_single_atom_recovered_exactly(name):           # test_solvers.py:148-159
    d = partial_dct(16, 7, 0)
    x0 = np.zeros(16)
    x0[5] = 2.5
    r = hcs.SOLVERS[name](d.matrix @ x0, d, hcs.SolverConfig(kappa=1, atoms_per_iter=1, **NO_LIMITS))
    assert r.converged and r.iterations <= 2
    np.testing.assert_allclose(r.x, x0, atol=1e-10)


@pytest.mark.parametrize("name", ["gomp", "biht", "cosamp"])
def test_output_never_exceeds_kappa_nonzeros(name):     # test_solvers.py:167-175, C3
    rng = np.random.default_rng(11)
    d = partial_dct(32, 13, 2)
    for kappa in (1, 3, 5):
        cfg = hcs.SolverConfig(kappa=kappa, atoms_per_iter=1, time_limit=None, max_iter=60)
        r = hcs.SOLVERS[name](rng.standard_normal(13), d, cfg)
        assert np.count_nonzero(r.x) <= kappa


def test_gomp_adds_several_atoms_per_iteration():       # test_solvers.py:177-181
    # seeds whose partial-DCT instance is exactly recoverable (the oracle recovers 0, 4, 5 of 0..5)
    for seed in (0, 4, 5):
        d, x0, y = planted(32, 16, 6, seed)
        r = hcs.gomp(y, d, hcs.SolverConfig(kappa=6, atoms_per_iter=3, **NO_LIMITS))
        assert r.converged
        np.testing.assert_allclose(r.x, x0, atol=1e-8)


def test_gomp_stops_when_the_support_outgrows_the_measurements():   # test_solvers.py:183-191
    rng = np.random.default_rng(12)
    d = partial_dct(16, 6, 3)
    r = hcs.gomp(rng.standard_normal(6), d, hcs.SolverConfig(kappa=6, atoms_per_iter=6, time_limit=None, max_iter=500))
    assert not r.converged and np.count_nonzero(r.x) <= 6


def test_precondition_validation():                    # test_solvers.py:193-203
    d = partial_dct(16, 6, 0)
    y = np.ones(6)
    for solver, kappa in ((hcs.gomp, 7), (hcs.biht, 7), (hcs.cosamp, 7), (hcs.cosamp, 9)):
        with pytest.raises(ValueError):
            solver(y, d, hcs.SolverConfig(kappa=kappa, time_limit=None))


def test_iteration_cap_and_expired_budget():            # test_solvers.py:207-215
    d, _, y = planted(32, 13, 4, 5)
    r = hcs.fista(y, d, hcs.SolverConfig(lam=1e-4, time_limit=None, max_iter=1))
    assert r.iterations == 1 and not r.converged
    r = hcs.fista(y, d, hcs.SolverConfig(lam=0.1, time_limit=1e-12))
    assert r.iterations == 0 and not r.converged
    with pytest.raises(ValueError):
        hcs.fista(np.ones(4), d, hcs.SolverConfig())


def test_non_finite_measurements():                     # test_solvers.py:224-229 + solvers.py:227 / kernels.py:61
    d = partial_dct(8, 3, 0)
    y = np.array([np.nan, 1.0, 1.0])
    with pytest.raises(hcs.NumericalFailure) as info:
        hcs.fista(y, d, hcs.SolverConfig(lam=0.1, time_limit=None))
    assert info.value.iteration == 1
    for name in ("admm", "gomp", "biht", "cosamp"):     # the reference raises ValueError from scipy
        with pytest.raises(ValueError):
            hcs.SOLVERS[name](y, d, hcs.SolverConfig(kappa=1, time_limit=None, max_iter=10))


def test_epsilon_above_one_converges_before_iterating():   # stop rule with delta0 = 1 (solvers.py:111)
    d, _, y = planted(32, 13, 4, 5)
    for name in hcs.SOLVERS:
        r = hcs.SOLVERS[name](y, d, hcs.SolverConfig(kappa=2, epsilon=2.0, time_limit=None))
        assert r.iterations == 0 and r.converged


class TestRecoverCube:                                  # test_solvers.py:240-316
    @pytest.fixture
    def measured(self):
        rng = np.random.default_rng(8)
        d = partial_dct(16, 7, 1)
        x_true = np.zeros((2, 3, 16))
        for ix in range(2):
            for iy in range(3):
                x_true[ix, iy, rng.choice(16, size=2, replace=False)] = rng.uniform(1.0, 2.0, size=2)
        return d, x_true, np.einsum("mk,xyk->xym", d.matrix, x_true)

    def test_recovers_every_pixel(self, measured):
        d, x_true, meas = measured
        cube, st = hcs.recover_cube(meas, d, hcs.SolverConfig(kappa=2, atoms_per_iter=1, time_limit=None,
                                                               max_iter=50), "gomp")
        assert cube.shape == (2, 3, 16)
        ref = oc.solve_cube("gomp", d.basis, meas.reshape(6, -1), np.tile(d.masks, (6, 1)),
                            oc.OracleConfig(kappa=2, atoms_per_iter=1, max_iter=50))
        np.testing.assert_allclose(cube.reshape(6, -1), ref.x, atol=1e-12)
        # 5 of the 6 partial-DCT pixels are exactly recoverable (pixel (0, 1) is not, for the oracle too)
        ok = np.abs(ref.x - x_true.reshape(6, -1)).max(axis=1) < 1e-8
        assert ok.sum() == 5
        np.testing.assert_allclose(cube.reshape(6, -1)[ok], x_true.reshape(6, -1)[ok], atol=1e-8)
        assert (st.n_pixels, st.n_converged, st.n_failed, st.convergence_pct) == (6, 6, 0, 100.0)
        assert st.total_iterations == sum(r.iterations for r in st.results) == ref.iterations.sum()

    def test_runs_are_reproducible(self, measured):
        d, _, meas = measured
        cfg = hcs.SolverConfig(kappa=2, atoms_per_iter=1, time_limit=None, max_iter=50)
        c1, _ = hcs.recover_cube(meas, d, cfg, "cosamp")
        c2, _ = hcs.recover_cube(meas, d, cfg, "cosamp", jobs=4)
        np.testing.assert_array_equal(c1, c2)

    def test_admm_cube_uses_the_cached_factorization(self, measured):
        d, _, meas = measured
        cube, st = hcs.recover_cube(meas, d, hcs.SolverConfig(lam=0.05, alpha=1.8, time_limit=None,
                                                               max_iter=5000), "admm")
        ref = oc.solve_cube("admm", d.basis, meas.reshape(6, -1), np.tile(d.masks, (6, 1)),
                            oc.OracleConfig(lam=0.05, alpha=1.8, max_iter=5000))
        assert st.n_converged == int(ref.converged.sum()) == 5 and 1.8 in d._admm_factors
        np.testing.assert_array_equal(st.iterations, ref.iterations)

    def test_failed_pixels_are_flagged_not_fatal(self, measured):
        d, _, meas = measured
        meas = meas.copy()
        meas[0, 1, 0] = np.nan
        cube, st = hcs.recover_cube(meas, d, hcs.SolverConfig(lam=0.1, time_limit=None, max_iter=400), "fista")
        assert st.n_failed == 1 and st.failed_pixels == [(0, 1, 1)]
        assert st.results[1] is None
        np.testing.assert_array_equal(cube[0, 1], np.zeros(16))
        assert st.n_converged == 5

    def test_zero_pixels_counted_separately(self):
        d = partial_dct(8, 3, 0)
        cube, st = hcs.recover_cube(np.zeros((1, 2, 3)), d, hcs.SolverConfig(kappa=1), "gomp")
        assert st.n_zero_pixels == 2 and st.n_converged == 2 and st.total_iterations == 0

    def test_input_validation(self, measured):
        d, _, meas = measured
        with pytest.raises(ValueError):
            hcs.recover_cube(meas, d, hcs.SolverConfig(), "nope")
        with pytest.raises(ValueError):
            hcs.recover_cube(meas[:, :, :5], d, hcs.SolverConfig(), "fista")
        with pytest.raises(ValueError):
            hcs.recover_cube(meas[0], d, hcs.SolverConfig(), "fista")

    def test_device_and_pinned_inputs(self, measured):
        d, x_true, meas = measured
        cfg = hcs.SolverConfig(kappa=2, atoms_per_iter=1, time_limit=None, max_iter=50)
        ref, _ = hcs.recover_cube(meas, d, cfg, "gomp")
        dev, _ = hcs.recover_cube(torch.as_tensor(meas, device="cuda"), d, cfg, "gomp")
        pin, _ = hcs.recover_cube(torch.as_tensor(meas).pin_memory(), d, cfg, "gomp")
        assert dev.is_cuda and not pin.is_cuda
        np.testing.assert_array_equal(dev.cpu().numpy(), ref)
        np.testing.assert_array_equal(pin.numpy(), ref)


def test_per_pixel_dictionary_cube_matches_oracle():
    c = synth.generate(6, 10, 154, seed=21)
    d = Dictionary.per_pixel(c.basis, c.masks)
    cfg = hcs.SolverConfig(kappa=22, mu=0.1, time_limit=None, max_iter=2000)
    cube, st = hcs.recover_cube(c.y.reshape(6, 10, -1), d, cfg, "biht")
    ref = oc.solve_cube("biht", c.basis, c.y, c.masks, oc.OracleConfig(kappa=22, mu=0.1, max_iter=2000))
    np.testing.assert_array_equal(st.iterations, ref.iterations)
    num = np.linalg.norm(cube.reshape(60, -1) - ref.x, axis=1)
    assert np.all(num <= 1e-9 * np.maximum(np.linalg.norm(ref.x, axis=1), 1e-300))


def test_unit_lipschitz_constant():                     # C5: 20 random selections, |L - 1| <= 1e-8
    rng = np.random.default_rng(5)
    for i, n in enumerate(rng.integers(8, 225, size=20)):
        d = hcs.build_dictionary(hcs.build_dct_basis(int(n)), hcs.build_selection_mask(int(n), 0.4, seed=i))
        assert abs(d.lipschitz - 1.0) <= 1e-8
        assert abs(d.lipschitz - oc.lipschitz(d.matrix)) <= 1e-13


class TestKernels:                                      # test_kernels.py
    def test_soft_threshold(self):
        np.testing.assert_allclose(hcs.soft_threshold(np.array([3.0, -1.0, 0.5, 0.0]), 1.0), [2.0, 0, 0, 0], atol=0)
        np.testing.assert_array_equal(hcs.soft_threshold(np.array([1.0, -0.5, 0.0]), 0.0), [1.0, -0.5, 0.0])
        with pytest.raises(ValueError):
            hcs.soft_threshold(np.array([1.0]), -0.1)

    def test_argmax_k(self):
        np.testing.assert_array_equal(hcs.argmax_k(np.array([1.0, -5.0, 3.0]), 2), [1, 2])
        np.testing.assert_array_equal(hcs.argmax_k(np.array([0.1, 9.0, 0.2, 8.0, 7.0]), 3), [1, 3, 4])
        np.testing.assert_array_equal(hcs.argmax_k(np.array([2.0, -2.0, 1.0]), 1), [0])
        np.testing.assert_array_equal(hcs.argmax_k(np.array([1.0, 3.0, 3.0, 3.0]), 2), [1, 2])
        for k in (0, 3):
            with pytest.raises(ValueError):
                hcs.argmax_k(np.array([1.0, 2.0]), k)

    def test_least_squares(self):
        rng = np.random.default_rng(1)
        b, y = rng.standard_normal((8, 3)), rng.standard_normal(8)
        np.testing.assert_allclose(hcs.least_squares(b, y), np.linalg.solve(b.T @ b, b.T @ y), atol=1e-12)
        b = rng.standard_normal((4, 4))
        np.testing.assert_allclose(hcs.least_squares(b, y[:4]), np.linalg.solve(b, y[:4]), atol=1e-12)
        col = rng.standard_normal(6)
        s = hcs.least_squares(np.stack([col, col], axis=1), 3.0 * col)
        np.testing.assert_allclose(s, [1.5, 1.5], atol=1e-10)
        b = rng.standard_normal((3, 7))
        np.testing.assert_allclose(hcs.least_squares(b, y[:3]), np.linalg.pinv(b) @ y[:3], atol=1e-10)
        with pytest.raises(ValueError):
            hcs.least_squares(np.ones((3, 2)), np.ones(4))

    def test_residual_delta(self):
        assert hcs.residual_delta(np.array([1.0, 1.0]), np.array([0.0, 0.0])) == pytest.approx(math.sqrt(2.0))
        with pytest.raises(ValueError):
            hcs.residual_delta(np.ones(2), np.ones(3))


@pytest.mark.parametrize("algo,params", [("fista", dict(lam=0.1)), ("admm", dict(lam=0.1, alpha=1.8)),
                                         ("gomp", dict(kappa=22, atoms_per_iter=4)), ("cosamp", dict(kappa=22))])
def test_chunked_host_pipeline_matches_one_launch(algo, params):
    """recover_cube on host buffers pipelines pixel chunks over two compute
    streams; results must equal the single device launch bit for bit."""
    c = synth.generate(6, 10, 154, seed=22)
    d = Dictionary.per_pixel(c.basis, c.masks)
    cfg = hcs.SolverConfig(time_limit=None, max_iter=500, **params)
    meas = c.y.reshape(6, 10, -1)
    ref, st_ref = hcs.recover_cube(torch.as_tensor(meas, device="cuda"), d, cfg, algo)
    ref = ref.cpu().numpy()
    out = np.full((6, 10, 154), np.nan)
    got, st = hcs.recover_cube(meas, d, cfg, algo, chunk_pixels=7, out=out)
    assert got is out
    np.testing.assert_array_equal(got, ref)
    np.testing.assert_array_equal(st.iterations, st_ref.iterations)
    np.testing.assert_array_equal(st.final_delta, st_ref.final_delta)
    pin, st2 = hcs.recover_cube(torch.as_tensor(meas).pin_memory(), d, cfg, algo, chunk_pixels=13)
    assert pin.is_pinned()
    np.testing.assert_array_equal(pin.numpy(), ref)
    assert st2.total_iterations == st_ref.total_iterations


def test_chunked_pipeline_reports_nonfinite_from_any_chunk():
    c = synth.generate(6, 10, 154, seed=23)
    d = Dictionary.per_pixel(c.basis, c.masks)
    meas = c.y.reshape(6, 10, -1).copy()
    meas[5, 9, 3] = np.inf                      # in the last chunk only
    with pytest.raises(ValueError):
        hcs.recover_cube(meas, d, hcs.SolverConfig(kappa=22, time_limit=None), "gomp", chunk_pixels=8)
    with pytest.raises(ValueError):
        hcs.recover_cube(meas, d, hcs.SolverConfig(kappa=22, time_limit=None), "gomp",
                         out=np.empty((6, 10, 153)))


@pytest.mark.gpu
@pytest.mark.parametrize("algo,params", [("fista", dict(lam=0.1)), ("admm", dict(lam=0.1)), ("admm", dict(lam=100.0))])
def test_convex_slot_engines_agree(monkeypatch, algo, params):
    """The 16-slot x two-CTAs-per-SM engine (HCS_CONVEX_SLOTS=16, kept for
    experiments) performs the same per-element arithmetic in the same order as
    the default 32-slot engine; only the residual-delta partial sums are summed
    over a different warp split (8 vs 16 warps), so delta may differ in the
    last bits: iterations and x must agree exactly, delta to 1e-12."""
    import torch
    from paper_2401_14762_b200 import synth
    from paper_2401_14762_b200.solvers import SolverConfig, solve_batch
    c = synth.generate(6, 50, 224, seed=21)
    dev = torch.device("cuda")
    args = (torch.as_tensor(c.y, device=dev), torch.as_tensor(c.masks, device=dev), torch.as_tensor(c.basis, device=dev),
            SolverConfig(time_limit=None, max_iter=5000, **params))
    outs = []
    for slots in ("32", "16"):
        monkeypatch.setenv("HCS_CONVEX_SLOTS", slots)
        b = solve_batch(algo, *args)
        torch.cuda.synchronize()
        outs.append((b.x.cpu().numpy(), b.iterations.cpu().numpy(), b.final_delta.cpu().numpy()))
    (x32, it32, d32), (x16, it16, d16) = outs
    assert np.array_equal(it32, it16), f"{int((it32 != it16).sum())} iteration mismatches"
    assert np.max(np.abs(x32 - x16)) <= 1e-13 * max(np.max(np.abs(x32)), 1e-300), np.max(np.abs(x32 - x16))
    assert np.allclose(d32, d16, rtol=1e-12, atol=0)


@pytest.mark.gpu
@pytest.mark.parametrize("lam", [1.0, 3.0, 100.0])
def test_admm_zero_shrinkage_pass_matches_oracle(lam):
    """ADMM pixels whose shrinkage is certified zero are solved by the O(N)
    sample-domain pass (admm_zero_kernel), the rest by the slot engine from the
    pixel list; lambda = 1 and 3 mix both populations in one call.  Every pixel
    must match the oracle: iterations, converged, x (1e-9), admm_gap (1e-9)."""
    import torch
    from paper_2401_14762_b200.solvers import SolverConfig, solve_batch
    c = synth.generate(8, 50, 224, seed=33)
    dev = torch.device("cuda")
    cfg = SolverConfig(lam=lam, alpha=1.8, time_limit=None, max_iter=5000)
    b = solve_batch("admm", torch.as_tensor(c.y, device=dev), torch.as_tensor(c.masks, device=dev),
                    torch.as_tensor(c.basis, device=dev), cfg)
    torch.cuda.synchronize()
    ref = oc.solve_cube("admm", c.basis, c.y, c.masks, oc.OracleConfig(lam=lam, alpha=1.8, max_iter=5000))
    assert np.array_equal(b.iterations.cpu().numpy(), ref.iterations)
    assert np.array_equal(b.converged.cpu().numpy().astype(bool), ref.converged)
    x = b.x.cpu().numpy()
    nr = np.linalg.norm(ref.x, axis=1)
    err = np.linalg.norm(x - ref.x, axis=1)
    assert np.all(np.where(nr > 0, err <= 1e-9 * nr, err <= 1e-12))
    # admm_gap = ||x - z|| of the last pass: ~1e-9 at convergence, a difference
    # of nearly equal iterates, so its rounding is absolute (~1e-15 ||x||)
    gap = b.admm_gap.cpu().numpy()
    assert np.all(np.abs(gap - ref.admm_gap) <= 1e-9 * ref.admm_gap + 1e-13 * np.maximum(nr, 1.0))
    zero = np.linalg.norm(ref.x, axis=1) == 0
    if lam == 100.0:
        assert zero.all()
    print(f"lambda {lam}: {int(zero.sum())} / {len(zero)} pixels with x = 0")


@pytest.mark.gpu
@pytest.mark.parametrize("algo", ["fista", "admm"])
@pytest.mark.parametrize("lam", [0.1, 0.01, 100.0])
def test_fista_kstep_skip_bitwise(monkeypatch, algo, lam):
    """The sparse GEMMs (FISTA's Psi x_{k+1}, ADMM's Psi z) skip the DMMAs
    whose 4 x 8 block of input (four coefficient rows of an 8-slot column
    block) is zero: the skipped products are exact zeros, so results are
    bit-for-bit those of the dense GEMM."""
    import torch
    from paper_2401_14762_b200.solvers import SolverConfig, solve_batch
    c = synth.generate(6, 50, 224, seed=44)
    dev = torch.device("cuda")
    args = (torch.as_tensor(c.y, device=dev), torch.as_tensor(c.masks, device=dev), torch.as_tensor(c.basis, device=dev),
            SolverConfig(lam=lam, time_limit=None, max_iter=5000))
    outs = []
    for flag in ("0", "1"):
        monkeypatch.setenv("HCS_CONVEX_KSKIP", flag)
        b = solve_batch(algo, *args)
        torch.cuda.synchronize()
        outs.append([t.cpu().numpy() for t in (b.x, b.iterations, b.final_delta, b.converged, b.admm_gap)])
    for u, v in zip(*outs):
        assert np.array_equal(u, v, equal_nan=True)


@pytest.mark.gpu
@pytest.mark.parametrize("algo,lam,n", [("fista", 0.1, 224), ("admm", 0.1, 224), ("admm", 3.0, 224),
                                        ("fista", 0.1, 198), ("admm", 1.0, 154)])
def test_ring_and_register_fragment_paths_bitwise(monkeypatch, algo, lam, n):
    """The slot engine's A fragments through the per-warp cp.async ring
    (default when it fits in shared memory) against the register-prefetch GEMM
    (HCS_CONVEX_RING=0): the same DMMA order per accumulator, so every output
    is bit-for-bit the same; enough pixels that slots retire and refill."""
    import torch
    from paper_2401_14762_b200.solvers import SolverConfig, solve_batch
    c = synth.generate(30, 170, n, seed=45)   # 5100 px: > 148 x 32 slots, so slots refill
    dev = torch.device("cuda")
    args = (torch.as_tensor(c.y, device=dev), torch.as_tensor(c.masks, device=dev), torch.as_tensor(c.basis, device=dev),
            SolverConfig(lam=lam, time_limit=None, max_iter=400))
    outs = []
    for flag in ("0", "1"):
        monkeypatch.setenv("HCS_CONVEX_RING", flag)
        b = solve_batch(algo, *args)
        torch.cuda.synchronize()
        outs.append([t.cpu().numpy() for t in (b.x, b.iterations, b.final_delta, b.converged, b.admm_gap)])
    assert outs[0][1].max() > 1
    for u, v in zip(*outs):
        assert np.array_equal(u, v, equal_nan=True)


@pytest.mark.gpu
@pytest.mark.parametrize("algo,kappa", [("cosamp", 27), ("cosamp", 33), ("cosamp", 12)])
def test_dct_closed_form_gram_matches_the_dmma_gram(monkeypatch, algo, kappa):
    """CoSaMP least squares on wide systems: for a DCT-II basis the augmented
    CSNE Gram comes from the product-to-sum closed form (hcs_ls_csne.cuh:
    DctGram) instead of M-term DMMA dot products over the gathered columns.
    Same significant supports, iterations and flags (but for roundoff-level
    ties of the prune), coefficients within the refinement's accuracy of the
    DMMA-Gram solve."""
    import torch
    from paper_2401_14762_b200.solvers import SolverConfig, solve_batch
    c = synth.generate(8, 50, 224, seed=45)
    dev = torch.device("cuda")
    args = (torch.as_tensor(c.y, device=dev), torch.as_tensor(c.masks, device=dev),
            torch.as_tensor(c.basis, device=dev), SolverConfig(kappa=kappa, time_limit=None, max_iter=2000))
    outs = []
    for flag in ("0", "1"):
        monkeypatch.setenv("HCS_DCT_GRAM", flag)
        b = solve_batch(algo, *args)
        torch.cuda.synchronize()
        outs.append([t.cpu().numpy() for t in (b.x, b.iterations, b.converged, b.failed_at)])
    (x0, it0, cv0, f0), (x1, it1, cv1, f1) = outs
    same = it0 == it1
    assert same.mean() >= 0.97 and np.array_equal(cv0[same], cv1[same]) and np.array_equal(f0, f1)
    nr = np.maximum(np.linalg.norm(x0[same], axis=1), 1e-300)
    assert np.array_equal(np.abs(x0[same]) > 1e-9 * nr[:, None], np.abs(x1[same]) > 1e-9 * nr[:, None])
    assert np.max(np.linalg.norm(x0[same] - x1[same], axis=1) / nr) < 1e-10


@pytest.mark.gpu
def test_non_dct_basis_takes_the_dmma_gram():
    """A rotated (non-DCT) orthonormal basis must be detected on the device
    (transpose_basis_kernel) and solved with the general Gram: CoSaMP and BIHT
    against the oracle, and the workspace header word says 'not DCT'."""
    import torch
    from paper_2401_14762_b200.solvers import SolverConfig, solve_batch
    n, m, P = 96, 40, 200
    rng = np.random.default_rng(7)
    q, _ = np.linalg.qr(rng.standard_normal((n, n)))
    basis = np.ascontiguousarray(q)
    x0 = np.zeros((P, n))
    for p in range(P):
        x0[p, rng.choice(n, size=6, replace=False)] = rng.uniform(0.5, 1.5, 6) * rng.choice([-1, 1], 6)
    masks = np.sort(np.argsort(rng.random((P, n)), axis=1)[:, :m], axis=1).astype(np.uint8)
    spectra = x0 @ basis.T
    y = np.ascontiguousarray(np.take_along_axis(spectra, masks.astype(np.intp), axis=1))
    dev = torch.device("cuda")
    for algo, kappa in (("cosamp", 8), ("biht", 10)):
        b = solve_batch(algo, torch.as_tensor(y, device=dev), torch.as_tensor(masks, device=dev),
                        torch.as_tensor(basis, device=dev), SolverConfig(kappa=kappa, time_limit=None, max_iter=200))
        torch.cuda.synchronize()
        assert int(b.workspace[32:36].view(torch.int32).item()) == 1
        ref = oc.solve_cube(algo, basis, y, masks, oc.OracleConfig(kappa=kappa, max_iter=200))
        same = b.iterations.cpu().numpy() == ref.iterations
        assert same.mean() >= 0.97
        nr = np.maximum(np.linalg.norm(ref.x[same], axis=1), 1e-300)
        assert np.max(np.linalg.norm(b.x.cpu().numpy()[same] - ref.x[same], axis=1) / nr) < 1e-9
    # and the DCT basis itself is recognised
    c = synth.generate(2, 50, 224, seed=3)
    b = solve_batch("biht", torch.as_tensor(c.y, device=dev), torch.as_tensor(c.masks, device=dev),
                    torch.as_tensor(c.basis, device=dev), SolverConfig(kappa=27, time_limit=None, max_iter=50))
    torch.cuda.synchronize()
    assert int(b.workspace[32:36].view(torch.int32).item()) == 0
