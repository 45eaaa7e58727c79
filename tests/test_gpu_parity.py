"""GPU parity: libhypercs_b200 vs the reference golden fixtures and the CPU oracle.

Bar (north_star / SURVEY.md §8(c)): coefficients within 1e-9 norm-relative
(FP64), identical significant supports, identical iteration counts and
convergence flags -- except tie exceptions (first divergent selection
roundoff-degenerate on the reference side), which are counted and capped.
"""

import json
import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import cpu_solvers as oc  # noqa: E402
from paper_2401_14762_b200 import synth  # noqa: E402
from paper_2401_14762_b200.solvers import SolverConfig, solve_batch  # noqa: E402
from parity import compare, load_traces  # noqa: E402

pytestmark = pytest.mark.gpu

CASES = [
    "cfg1_gomp_k24", "cfg2_fista_l100", "cfg2_admm_l100", "cfg2_fista_l0.1", "cfg2_admm_l0.1",
    "cfg3_biht_k22", "cfg3_gomp_k22", "cfg4_cosamp_k33", "cfg5_cosamp_k27", "cfg5_gomp_k27",
    "cfg5_gomp_k33", "cfg5_biht_k27", "cfg5_biht_k33",
]
TRACE_CALLS = 64


def decode_trace(tr, n):
    """(P, calls, 4) int64 bitmaps + lengths -> per-pixel lists of (k, picks)."""
    tr_np = tr[0].cpu().numpy().view(np.uint64)
    lens = tr[1].cpu().numpy()
    out = []
    for p in range(tr_np.shape[0]):
        calls = []
        for c in range(min(int(lens[p]), tr_np.shape[1])):
            bits = np.unpackbits(tr_np[p, c].view(np.uint8), bitorder="little")
            idx = tuple(int(i) for i in np.flatnonzero(bits))
            calls.append((len(idx), idx))
        out.append(calls)
    return out


def run_gpu(algo, y, masks, basis, cfg, trace=False):
    dev = torch.device("cuda")
    b = solve_batch(algo, torch.as_tensor(np.ascontiguousarray(y), device=dev),
                    torch.as_tensor(np.ascontiguousarray(masks, dtype=np.uint8), device=dev),
                    torch.as_tensor(basis, device=dev), cfg, trace_calls=TRACE_CALLS if trace else 0)
    torch.cuda.synchronize()
    res = dict(x=b.x.cpu().numpy(), iterations=b.iterations.cpu().numpy(),
               converged=b.converged.cpu().numpy().astype(bool), failed_at=b.failed_at.cpu().numpy(),
               final_delta=b.final_delta.cpu().numpy(), admm_gap=b.admm_gap.cpu().numpy(),
               lipschitz=b.lipschitz.cpu().numpy())
    if trace:
        res["trace"] = decode_trace((b.trace, b.trace_len), basis.shape[0])
    return res


def make_replay(algo, basis, y, masks, ocfg):
    """Forced-selection replay of SURVEY.md §8(c) through the oracle."""
    def replay(p, force):
        rec = oc.Recorder(force=force, ynorm=float(np.linalg.norm(np.nan_to_num(y[p]))))
        return oc.solve_pixel(algo, y[p], basis[np.asarray(masks[p]).astype(np.intp), :], ocfg, trace=rec)
    return replay


def load_case(golden_dir, name):
    z = np.load(golden_dir / f"{name}.npz", allow_pickle=False)
    return z, json.loads(str(z["meta"]))


@pytest.mark.parametrize("name", CASES)
def test_gpu_matches_reference_golden(golden_dir, name):
    z, meta = load_case(golden_dir, name)
    algo = meta["algo"]
    basis = synth.dct_basis(int(z["n"]))
    cfg = SolverConfig(time_limit=None, max_iter=meta["max_iter"], **meta["params"])
    greedy = algo in ("gomp", "biht", "cosamp")
    got = run_gpu(algo, z["y"], z["masks"], basis, cfg, trace=greedy)
    ref = dict(x=z["x"], iterations=z["iterations"], converged=z["converged"], failed_at=z["failed_at"])
    ocfg = oc.OracleConfig(max_iter=meta["max_iter"] or 0, **meta["params"])
    rep = compare(ref, got, z["y"], load_traces(z["traces"]) if greedy else None,
                  got.get("trace"), algo, replay=make_replay(algo, basis, z["y"], z["masks"], ocfg))
    print(json.dumps({k: v for k, v in rep.items() if k != "bad"}, default=str)[:400])
    assert not rep["bad"], rep
    assert len(rep["ties"]) <= 2, rep
    ok = z["failed_at"] < 0
    if algo == "fista":
        np.testing.assert_allclose(got["lipschitz"], z["lipschitz"], rtol=0, atol=1e-13)
    same = ok & (z["iterations"] == got["iterations"])
    floor = 1e-12 * np.linalg.norm(np.nan_to_num(z["y"]), axis=1)[same]
    assert np.all(np.abs(got["final_delta"][same] - z["final_delta"][same])
                  <= 1e-6 * np.abs(z["final_delta"][same]) + floor)
    if algo == "admm":
        g = same & ~np.isnan(z["admm_gap"])
        np.testing.assert_allclose(got["admm_gap"][g], z["admm_gap"][g], rtol=1e-6, atol=1e-12)


# larger seeded cubes against the oracle (run here on the GPU box's CPU)
ORACLE_CASES = [
    ("jasper", "gomp", dict(kappa=24, atoms_per_iter=4), None, 600),
    # gOMP with |S| > kappa after one pass: least-squares systems of 24..60 columns
    # (warp kernel pre-columns) and, past 64 columns, the CTA kernel's spill path
    ("salinas", "gomp", dict(kappa=12, atoms_per_iter=12), 6, 200),
    ("jasper", "fista", dict(lam=0.1), 5000, 200),
    ("jasper", "admm", dict(lam=0.1, alpha=1.8), 5000, 120),
    ("jasper", "fista", dict(lam=100.0), 5000, 400),
    ("jasper", "admm", dict(lam=100.0, alpha=1.8), 5000, 300),
    ("china", "biht", dict(kappa=22, mu=0.1), 2000, 500),
    ("china", "gomp", dict(kappa=22, atoms_per_iter=4), None, 500),
    ("salinas", "cosamp", dict(kappa=33), 2000, 500),
    ("salinas", "cosamp", dict(kappa=27), 2000, 300),
    ("salinas", "biht", dict(kappa=33, mu=0.1), 2000, 300),
]


@pytest.mark.parametrize("cube,algo,params,cap,npix", ORACLE_CASES)
def test_gpu_matches_oracle(cube, algo, params, cap, npix):
    n = synth.CUBES[cube]["n"]
    c = synth.generate(npix // 20, 20, n, seed=7 + npix)
    cfg = SolverConfig(time_limit=None, max_iter=cap, **params)
    greedy = algo in ("gomp", "biht", "cosamp")
    got = run_gpu(algo, c.y, c.masks, c.basis, cfg, trace=greedy)
    ocfg = oc.OracleConfig(max_iter=cap or 0, **params)
    ref = oc.solve_cube(algo, c.basis, c.y, c.masks, ocfg, jobs=8, trace=greedy)
    refd = dict(x=ref.x, iterations=ref.iterations, converged=ref.converged, failed_at=ref.failed_at)
    rep = compare(refd, got, c.y, ref.traces, got.get("trace"), algo,
                  replay=make_replay(algo, c.basis, c.y, c.masks, ocfg))
    print(json.dumps({k: (v if k != "ties" else v[:5]) for k, v in rep.items() if k != "bad"}, default=str)[:600])
    assert not rep["bad"], rep["bad"][:5]
    assert len(rep["ties"]) <= max(2, int(0.02 * npix)), rep["ties"][:5]
    # PSNR of the recovered spectra (metrics.py:30-55): within 0.01 dB outside the roundoff regime
    f_ref = ref.x @ c.basis.T
    f_gpu = got["x"] @ c.basis.T
    peak = np.abs(c.spectra).max()
    mse_r = np.mean((c.spectra - f_ref) ** 2)
    mse_g = np.mean((c.spectra - f_gpu) ** 2)
    p_r = 10 * math.log10(peak ** 2 / mse_r)
    p_g = 10 * math.log10(peak ** 2 / mse_g)
    if p_r < 200 and not rep["ties"]:
        assert abs(p_r - p_g) <= 0.01, (p_r, p_g)


def test_kernel_goldens(golden_dir):
    from paper_2401_14762_b200 import kernels as gk
    k = np.load(golden_dir / "kernels.npz")
    for i in range(4):
        np.testing.assert_array_equal(gk.soft_threshold(k["soft_v"], float(k[f"soft_t{i}"])), k[f"soft_out{i}"])
    for kk in (1, 4, 22, 66, 200):
        np.testing.assert_array_equal(gk.argmax_k(k["argk_v"], kk), k[f"argk_out{kk}"])
    for i in range(int(k["ls_count"])):
        s = gk.least_squares(k[f"ls_b{i}"], k[f"ls_y{i}"])
        ref = k[f"ls_s{i}"]
        np.testing.assert_allclose(s, ref, rtol=0, atol=1e-10 * max(1.0, np.abs(ref).max()))


def test_cosamp_cycling_tail_pixels():
    """CoSaMP pixels that never converge enter exact 2- and 4-cycles; the GPU
    skips whole periods (hcs_greedy.cu) and must still match the oracle's
    2000-iteration result exactly in x, delta, iterations and flags."""
    c = synth.generate(30, 100, 224, seed=11)
    pick = np.array([95, 711, 757, 1068, 1297, 1984, 2086, 2149, 2213, 2543, 0, 1, 2, 3])
    y, masks = c.y[pick], c.masks[pick]
    cfg = SolverConfig(kappa=27, time_limit=None, max_iter=2000)
    got = run_gpu("cosamp", y, masks, c.basis, cfg, trace=True)
    ref = oc.solve_cube("cosamp", c.basis, y, masks, oc.OracleConfig(kappa=27, max_iter=2000), jobs=8,
                        chunk=1, trace=True)
    assert (ref.iterations[:10] == 2000).all() and not ref.converged[:10].any()
    refd = dict(x=ref.x, iterations=ref.iterations, converged=ref.converged, failed_at=ref.failed_at)
    rep = compare(refd, got, y, ref.traces, got.get("trace"), "cosamp",
                  replay=make_replay("cosamp", c.basis, y, masks, oc.OracleConfig(kappa=27, max_iter=2000)))
    assert not rep["bad"], rep["bad"]
    np.testing.assert_allclose(got["final_delta"], ref.final_delta, rtol=1e-6, atol=1e-12)
