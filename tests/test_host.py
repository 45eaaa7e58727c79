"""Host-side logic (no GPU): config validation, stop rule, dictionaries,
generator, parity comparator.  Mirrors hypercs' test_solvers.py:28-89 and
test_transform.py semantics for the parts that run on the host."""

import math

import numpy as np
import pytest

from paper_2401_14762_b200 import synth
from paper_2401_14762_b200.solvers import SolverConfig, SolverState, StopDecision, lasso_objective, stop_check
from paper_2401_14762_b200.transform import Dictionary, build_dictionary, build_selection_mask, measure
from parity import compare, degenerate, first_divergence


class TestSolverConfig:      # test_solvers.py:28-62
    def test_defaults(self):
        cfg = SolverConfig()
        assert (cfg.lam, cfg.kappa, cfg.atoms_per_iter, cfg.mu, cfg.alpha, cfg.epsilon, cfg.time_limit,
                cfg.max_iter, cfg.seed) == (0.1, 1, 1, 0.1, 1.8, 1e-8, 2.0, None, 0)

    def test_atoms_per_iter_defaults_to_a_fifth_of_kappa(self):
        assert SolverConfig(kappa=18).atoms_per_iter == 3
        assert SolverConfig(kappa=24).atoms_per_iter == 4
        assert SolverConfig(kappa=27).atoms_per_iter == 5
        assert SolverConfig(kappa=33).atoms_per_iter == 6
        assert SolverConfig(kappa=4).atoms_per_iter == 1

    @pytest.mark.parametrize("kw", [dict(lam=-1.0), dict(kappa=0), dict(kappa=3, atoms_per_iter=4), dict(mu=0.0),
                                    dict(alpha=-0.5), dict(epsilon=0.0), dict(time_limit=0.0), dict(max_iter=0)])
    def test_validation(self, kw):
        with pytest.raises(ValueError):
            SolverConfig(**kw)

    def test_native_params(self):
        p = SolverConfig(lam=0.5, kappa=27, max_iter=None, time_limit=None).to_native()
        assert p.kappa == 27 and p.atoms_per_iter == 5 and p.max_iter == 0 and p.time_limit == 0.0


class TestStopRule:          # test_solvers.py:65-89
    def test_precedence(self):
        cfg = SolverConfig(epsilon=1e-2, time_limit=1.0, max_iter=5)
        assert stop_check(SolverState(np.zeros(2), delta=1e-3, iterations=99), cfg, 50.0) is StopDecision.CONVERGED
        cfg = SolverConfig(epsilon=1e-8, time_limit=1.0, max_iter=5)
        assert stop_check(SolverState(np.zeros(2), delta=1.0, iterations=99), cfg, 1.0) is StopDecision.TIMEOUT
        cfg = SolverConfig(epsilon=1e-8, time_limit=None, max_iter=5)
        assert stop_check(SolverState(np.zeros(2), delta=1.0, iterations=5), cfg, 0.0) is StopDecision.ITER_CAP

    def test_convergence_is_strict(self):
        cfg = SolverConfig(epsilon=1e-8, time_limit=None)
        assert stop_check(SolverState(np.zeros(2), delta=1e-8), cfg, 0.0) is StopDecision.CONTINUE


def test_lasso_objective_hand_value():    # test_solvers.py:92-101
    d = Dictionary.from_matrix(np.eye(2))
    assert lasso_objective(np.array([1.0, -2.0]), np.zeros(2), d, 0.5) == pytest.approx(4.0)


class TestDictionaries:
    def test_dct_basis_is_orthonormal(self):
        for n in (154, 198, 224):
            b = synth.dct_basis(n)
            assert np.abs(b.T @ b - np.eye(n)).max() < 1e-13

    def test_from_matrix_completes_orthonormal_rows(self):
        b = synth.dct_basis(32)
        rows = b[[1, 4, 9, 17], :]
        d = Dictionary.from_matrix(rows)
        np.testing.assert_allclose(d.matrix, rows, atol=0)
        assert np.abs(d.basis.T @ d.basis - np.eye(32)).max() < 1e-12
        assert d.m == 4 and d.n == 32

    def test_from_matrix_rejects_non_orthonormal(self):
        with pytest.raises(ValueError):
            Dictionary.from_matrix(np.random.default_rng(0).standard_normal((5, 12)))
        with pytest.raises(ValueError):
            Dictionary.from_matrix(np.eye(3) * (1 + 1j))

    def test_per_pixel_masks(self):
        b = synth.dct_basis(16)
        masks = np.array([[0, 3, 5], [1, 2, 15]])
        d = Dictionary.per_pixel(b, masks)
        assert not d.shared and d.n_pixels == 2 and d.m == 3
        np.testing.assert_array_equal(d.matrix_of(1), b[[1, 2, 15], :])
        with pytest.raises(ValueError):
            Dictionary.per_pixel(b, np.array([[3, 1, 2]]))        # not increasing
        with pytest.raises(ValueError):
            Dictionary.per_pixel(b, np.array([[0, 1, 16]]))       # out of range

    def test_admm_factor_is_cached_and_exact(self):
        b = synth.dct_basis(24)
        mask = build_selection_mask(24, 0.4, 3)
        d = build_dictionary(b, mask, alpha=1.8)
        assert 1.8 in d._admm_factors
        f = d.admm_factor(1.8)
        a = d.matrix
        rhs = np.random.default_rng(1).standard_normal(24)
        np.testing.assert_allclose(f.solve(rhs), np.linalg.solve(a.T @ a + 1.8 * np.eye(24), rhs), atol=1e-12)

    def test_selection_mask_rule(self):          # transform.py:122-136, test_transform.py:131-175
        m = build_selection_mask(224, 0.4, 0)
        assert m.m == 90 and np.all(np.diff(m.indices) > 0)
        assert build_selection_mask(198, 0.4, 0).m == 79 and build_selection_mask(154, 0.4, 0).m == 62
        np.testing.assert_array_equal(build_selection_mask(50, 0.5, 7).indices,
                                      build_selection_mask(50, 0.5, 7).indices)
        f = np.arange(224.0)
        np.testing.assert_array_equal(measure(f, m), m.indices.astype(float))


class TestGenerator:
    def test_shapes_and_sparsity(self):
        c = synth.generate(6, 5, 198, seed=2)
        assert c.y.shape == (30, 79) and c.masks.shape == (30, 79) and c.coeffs.shape == (30, 198)
        assert np.all(np.diff(c.masks.astype(int), axis=1) > 0)
        nz = (c.coeffs != 0).sum(axis=1)
        assert nz.min() >= 1 and nz.mean() < 30
        np.testing.assert_allclose(c.spectra, c.coeffs @ c.basis.T, atol=1e-12)
        np.testing.assert_array_equal(c.y, np.take_along_axis(c.spectra, c.masks.astype(np.intp), 1))
        mag = np.abs(c.coeffs)
        kept = mag[mag > 0]
        assert np.all(kept >= 0.1 * np.repeat(mag.max(axis=1), (mag > 0).sum(axis=1)) - 1e-15)

    def test_deterministic_tiling_and_slabs(self):
        a = synth.generate(8, 6, 40, seed=5, tiles=(2, 3))
        b = synth.generate(8, 6, 40, seed=5, tiles=(2, 3), x_range=(3, 8), workers=2)
        np.testing.assert_array_equal(a.y.reshape(8, 6, -1)[3:], b.y.reshape(5, 6, -1))
        assert a.seeds == tuple(range(5, 11))


class TestComparator:
    def test_tie_classification(self):
        ref = dict(x=np.array([[1.0, 0.0], [1.0, 0.0]]), iterations=np.array([2, 3]),
                   converged=np.array([True, True]), failed_at=np.array([-1, -1]))
        cand = dict(x=np.array([[1.0, 0.0], [1.0, 0.0]]), iterations=np.array([2, 4]),
                    converged=np.array([True, True]), failed_at=np.array([-1, -1]))
        y = np.ones((2, 2))
        tr_ref = [[[1, [0], 1.0, 0.5]], [[1, [0], 1.0, 0.5], [1, [1], 1e-16, 0.0]]]
        tr_cand = [[(1, (0,))], [(1, (0,)), (1, (0,))]]
        rep = compare(ref, cand, y, tr_ref, tr_cand)
        assert not rep["bad"] and len(rep["ties"]) == 1 and rep["ties"][0]["call"] == 1
        # a divergence at a well-separated selection is a real mismatch
        tr_ref[1][1] = [1, [1], 1.0, 0.3]
        rep = compare(ref, cand, y, tr_ref, tr_cand)
        assert len(rep["bad"]) == 1

    def test_forced_selection_replay(self):
        from oracle import cpu_solvers as oc
        v = np.array([1.0, 1e-20, 2e-20, 0.5])
        rec = oc.Recorder(force={0: (0, 1)}, ynorm=1.0)
        # k = 2: the 2nd/3rd magnitudes (0.5 vs 2e-20) are well separated: not forced
        assert tuple(oc.argmax_k(v, 2, rec)) == (0, 3) and rec.forced == 0
        rec = oc.Recorder(force={0: (2,)}, ynorm=1e13)
        # k = 1 with ||y|| = 1e13: max|v| = 1 <= 1e-12 * 1e13 is degenerate: forced
        assert tuple(oc.argmax_k(v, 1, rec)) == (2,) and rec.forced == 1

    def test_helpers(self):
        assert first_divergence([[1, [0]]], [(1, (0,))]) is None
        assert first_divergence([[1, [0]], [1, [2]]], [(1, (0,)), (1, (3,))]) == 1
        assert degenerate((1, (0,), 1e-14, 0.5), 1.0) and not degenerate((1, (0,), 1.0, 0.5), 1.0)
        assert math.isfinite(1.0)
