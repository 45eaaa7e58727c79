"""Pin the CPU oracle (oracle/cpu_solvers.py) to the reference's own outputs.

The fixtures in tests/golden/ were produced by the unmodified reference
(tests/golden/make_golden.py); these tests run without a GPU.
"""

import json

import numpy as np
import pytest

from oracle import cpu_solvers as oc
from paper_2401_14762_b200 import synth
from parity import compare, load_traces

CASES = [
    "cfg1_gomp_k24", "cfg2_fista_l100", "cfg2_admm_l100", "cfg2_fista_l0.1", "cfg2_admm_l0.1",
    "cfg3_biht_k22", "cfg3_gomp_k22", "cfg4_cosamp_k33", "cfg5_cosamp_k27", "cfg5_gomp_k27",
    "cfg5_gomp_k33", "cfg5_biht_k27", "cfg5_biht_k33",
]


def load_case(golden_dir, name):
    z = np.load(golden_dir / f"{name}.npz", allow_pickle=False)
    meta = json.loads(str(z["meta"]))
    return z, meta


def oracle_config(meta):
    p = dict(meta["params"])
    return oc.OracleConfig(max_iter=meta["max_iter"] or 0, **p)


@pytest.mark.parametrize("name", CASES)
def test_oracle_matches_reference_golden(golden_dir, name):
    z, meta = load_case(golden_dir, name)
    basis = synth.dct_basis(int(z["n"]))
    cfg = oracle_config(meta)
    got = oc.solve_cube(meta["algo"], basis, z["y"], z["masks"], cfg, trace=True)
    ref = dict(x=z["x"], iterations=z["iterations"], converged=z["converged"], failed_at=z["failed_at"])
    cand = dict(x=got.x, iterations=got.iterations, converged=got.converged, failed_at=got.failed_at)
    rep = compare(ref, cand, z["y"], load_traces(z["traces"]),
                  [[list(e[:2]) + list(e[2:]) for e in t] for t in got.traces], meta["algo"])
    assert not rep["bad"], rep
    # tie exceptions must stay rare (<= ~1.3%); 48 px -> at most 2
    assert len(rep["ties"]) <= 2, rep
    np.testing.assert_allclose(got.lipschitz, z["lipschitz"], rtol=0, atol=1e-13)
    # final delta / admm gap: relative 1e-6, absolute at the roundoff floor 1e-12 ||y||
    same = (z["failed_at"] < 0) & (z["iterations"] == got.iterations)
    floor = 1e-12 * np.linalg.norm(np.nan_to_num(z["y"]), axis=1)[same]
    assert np.all(np.abs(got.final_delta[same] - z["final_delta"][same])
                  <= 1e-6 * np.abs(z["final_delta"][same]) + floor)
    if meta["algo"] == "admm":
        g_ok = same & ~np.isnan(z["admm_gap"])
        np.testing.assert_allclose(got.admm_gap[g_ok], z["admm_gap"][g_ok], rtol=1e-6, atol=1e-12)


def test_golden_edge_cases_are_present(golden_dir):
    z, meta = load_case(golden_dir, "cfg2_fista_l0.1")
    # all-zero pixel: 0 iterations, converged, delta 0 (solvers.py:145-152)
    assert z["iterations"][3] == 0 and z["converged"][3] and z["final_delta"][3] == 0.0
    # NaN pixel fails at iteration 1 (test_solvers.py:224-229)
    assert z["failed_at"][5] == 1
    z, meta = load_case(golden_dir, "cfg2_admm_l0.1")
    assert meta["nan_error"] == "ValueError"      # cho_solve's chkfinite, solvers.py:227


def test_kernel_fixtures(golden_dir):
    k = np.load(golden_dir / "kernels.npz")
    for i in range(4):
        np.testing.assert_array_equal(oc.soft_threshold(k["soft_v"], float(k[f"soft_t{i}"])), k[f"soft_out{i}"])
    for kk in (1, 4, 22, 66, 200):
        np.testing.assert_array_equal(oc.argmax_k(k["argk_v"], kk), k[f"argk_out{kk}"])
    for i in range(int(k["ls_count"])):
        s = oc.least_squares(k[f"ls_b{i}"], k[f"ls_y{i}"])
        np.testing.assert_allclose(s, k[f"ls_s{i}"], rtol=0, atol=1e-10 * max(1.0, np.abs(k[f"ls_s{i}"]).max()))
    for n, seed, lip in k["lip_table"]:
        n, seed = int(n), int(seed)
        basis = synth.dct_basis(n)
        mask = np.sort(np.random.default_rng(seed).choice(n, synth.measured_count(n), replace=False))
        assert abs(oc.lipschitz(basis[mask, :]) - lip) <= 1e-13


def test_oracle_sparsify_matches_reference_golden(golden_dir):
    """oracle.sparsify vs hypercs.transform.sparsify (transform.py:73-97) outputs
    recorded by tests/golden/make_sparsify_golden.py: bit-identical kept vectors
    and statistics."""
    z = np.load(golden_dir / "sparsify.npz")
    for x, f, out, mean, std, zf in zip(z["x"], z["factor"], z["out"], z["mean"], z["std"], z["zero_fraction"]):
        o, m, s, zz = oc.sparsify(x, float(f))
        assert np.array_equal(o, out)
        assert m == mean and s == std and zz == zf
    with pytest.raises(ValueError):
        oc.sparsify(np.array([1.0]), -0.5)
    with pytest.raises(ValueError):
        oc.sparsify(np.array([]), 0.1)
