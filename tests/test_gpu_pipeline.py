"""GPU stages over a run directory: synth -> recover ->
report, per-pixel masks through HSM2, a shared mask through the reference's
HSM1, and the CLI's exit codes (cli.py:46-49)."""

import csv
import json

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import cpu_solvers as oc  # noqa: E402
from paper_2401_14762_b200 import pipeline as pl  # noqa: E402
from paper_2401_14762_b200 import synth  # noqa: E402
from paper_2401_14762_b200.solvers import SolverConfig, solve_batch  # noqa: E402

pytestmark = pytest.mark.gpu


def test_synth_recover_report_per_pixel(tmp_path):
    run = tmp_path / "run"
    pl.run_synth(run, cube="jasper", seed=0, x_range=(0, 6))
    meas, n, masks = pl.load_measurements(run / pl.MEASUREMENTS_FILE)
    assert meas.shape == (6, 100, 79) and n == 198 and masks.shape == meas.shape
    cfg = SolverConfig(kappa=24, atoms_per_iter=4, time_limit=None)
    stats, tag = pl.run_recover(run, "gomp", cfg)
    assert tag == "gomp_kappa24"
    spectra = np.load(run / f"recovered_{tag}.npy")
    # the same recovery through solve_batch, and the oracle on a few pixels
    basis = synth.dct_basis(n)
    dev = torch.device("cuda")
    b = solve_batch("gomp", torch.as_tensor(meas.reshape(-1, 79), device=dev),
                    torch.as_tensor(masks.reshape(-1, 79), device=dev), torch.as_tensor(basis, device=dev), cfg)
    x = b.x.cpu().numpy()
    np.testing.assert_allclose(spectra.reshape(-1, n), x @ basis.T, rtol=0, atol=1e-12)
    assert stats.total_iterations == int(b.iterations.sum())
    ref = oc.solve_cube("gomp", basis, meas.reshape(-1, 79)[:40], masks.reshape(-1, 79)[:40],
                        oc.OracleConfig(kappa=24, atoms_per_iter=4))
    rel = np.linalg.norm(x[:40] - ref.x, axis=1) / np.maximum(np.linalg.norm(ref.x, axis=1), 1e-300)
    assert np.max(rel) < 1e-9
    meta = json.loads((run / f"run_{tag}.json").read_text())
    assert meta["n_pixels"] == 600 and meta["param_label"] == "κ=24"
    with open(run / f"pixels_{tag}.csv") as fh:
        rows = list(csv.reader(fh))
    assert rows[0] == ["x", "y", "iterations", "converged", "elapsed_s", "final_delta", "failed"]
    assert len(rows) == 601 and rows[101][:2] == ["1", "0"]          # x-major order (divmod(index, y))
    pl.run_recover(run, "fista", SolverConfig(lam=0.1, max_iter=5000, time_limit=None))
    rep = pl.run_report(run)
    assert sorted(r.algorithm for r in rep) == ["fista", "gomp"]
    ref_spectra = np.load(run / pl.SPARSIFIED_FILE)
    g = [r for r in rep if r.algorithm == "gomp"][0]
    peak = np.max(np.abs(ref_spectra))
    mse = np.mean((ref_spectra - spectra) ** 2)
    assert abs(g.psnr_db - 10 * np.log10(peak * peak / mse)) < 1e-9
    assert pl.read_report(run / pl.REPORT_FILE)[0].dataset == "synthetic-jasper"


def test_shared_mask_hsm1_run(tmp_path):
    """The reference's own layout: one mask for the cube, HSM1 complex payload."""
    run = tmp_path / "run"
    run.mkdir()
    c = synth.generate(4, 25, 154, seed=3)
    idx = np.sort(np.random.default_rng(1).choice(154, 62, replace=False))
    f = c.spectra.reshape(4, 25, 154)
    np.save(run / pl.SPARSIFIED_FILE, f)
    pl.save_measurements(run / pl.MEASUREMENTS_FILE, f[:, :, idx], 154)
    pl.save_mask(run / pl.MASK_FILE, 154, 1, indices=idx)
    cfg = SolverConfig(kappa=22, mu=0.1, max_iter=2000, time_limit=None)
    stats, tag = pl.run_recover(run, "biht", cfg)
    basis = synth.dct_basis(154)
    y = f[:, :, idx].reshape(-1, 62)
    ref = oc.solve_cube("biht", basis, y, np.tile(idx.astype(np.uint8), (100, 1)), oc.OracleConfig(kappa=22, mu=0.1,
                                                                                                   max_iter=2000))
    spectra = np.load(run / f"recovered_{tag}.npy").reshape(-1, 154)
    np.testing.assert_allclose(spectra, ref.x @ basis.T, rtol=0, atol=1e-9)
    assert stats.total_iterations == int(ref.iterations.sum())


def test_cli_bench_chain_and_exit_codes(tmp_path):
    out = tmp_path / "bench"
    rc = pl.main(["bench", "--out", str(out), "--cube", "china", "--rows", "2", "--algorithm", "cosamp,admm",
                  "--kappa", "22", "--lam", "100", "--max-iter", "2000"])
    assert rc == pl.EXIT_OK
    rows = pl.read_report(out / pl.REPORT_FILE)
    assert [(r.algorithm, r.param_label) for r in rows] == [("admm", "λ=100"), ("cosamp", "κ=22")]
    # mask / measurement mismatch: file-format error
    pl.save_mask(out / pl.MASK_FILE, 154, 0, m=61)
    assert pl.main(["recover", "--input", str(out), "--algorithm", "gomp", "--kappa", "5"]) == pl.EXIT_IO
