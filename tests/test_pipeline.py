"""Run-directory formats and report rows, host side.

Pinned to files written by the reference's own writers
(tests/golden/make_format_golden.py: cli.save_measurements, transform.save_mask,
metrics.write_report): the pipeline reads them and writes byte-identical ones.
The per-pixel extension (HSM2, ``indices=per-pixel``) round-trips.  The GPU
stages (synth / recover / report over a run directory) are in
tests/test_gpu_pipeline.py.
"""

import json
import math
from pathlib import Path

import numpy as np
import pytest

from paper_2401_14762_b200 import pipeline as pl
from paper_2401_14762_b200.solvers import SolverConfig

GOLD = Path(__file__).resolve().parent / "golden" / "formats"


def _inputs():
    return json.loads((GOLD / "inputs.json").read_text())


def test_reads_reference_hsm1():
    meas, n, masks = pl.load_measurements(GOLD / "ref_measurements.hsm")
    inp = _inputs()
    assert n == inp["n"] and masks is None
    np.testing.assert_array_equal(meas, np.array(inp["measurements"]))


def test_writes_reference_hsm1_bytes(tmp_path):
    inp = _inputs()
    pl.save_measurements(tmp_path / "m.hsm", np.array(inp["measurements"]), inp["n"])
    assert (tmp_path / "m.hsm").read_bytes() == (GOLD / "ref_measurements.hsm").read_bytes()


def test_mask_text_matches_reference(tmp_path):
    inp = _inputs()["mask"]
    mk = pl.load_mask(GOLD / "ref_mask.txt")
    assert mk["n"] == inp["n"] and mk["seed"] == inp["seed"] and mk["m"] == len(inp["indices"])
    assert mk["indices"].tolist() == inp["indices"]
    pl.save_mask(tmp_path / "mask.txt", inp["n"], inp["seed"], indices=inp["indices"])
    assert (tmp_path / "mask.txt").read_bytes() == (GOLD / "ref_mask.txt").read_bytes()


def test_hsm2_per_pixel_round_trip(tmp_path):
    rng = np.random.default_rng(0)
    x, y, m, n = 4, 3, 7, 20
    meas = rng.standard_normal((x, y, m))
    masks = np.sort(np.argsort(rng.random((x * y, n)), axis=1)[:, :m], axis=1).astype(np.uint8).reshape(x, y, m)
    pl.save_measurements(tmp_path / "m.hsm", meas, n, masks=masks)
    got, n2, masks2 = pl.load_measurements(tmp_path / "m.hsm")
    assert n2 == n
    np.testing.assert_array_equal(got, meas)
    np.testing.assert_array_equal(masks2, masks)
    raw = (tmp_path / "m.hsm").read_bytes()
    assert raw[:4] == b"HSM2" and len(raw) == 4 + 20 + x * y * m * 9
    pl.save_mask(tmp_path / "mask.txt", n, 3, m=m)
    mk = pl.load_mask(tmp_path / "mask.txt")
    assert mk == dict(seed=3, n=n, m=m, indices=None)


def test_measurement_file_errors(tmp_path):
    p = tmp_path / "bad.hsm"
    p.write_bytes(b"HSC1" + bytes(16))
    with pytest.raises(pl.PipelineFileError):
        pl.load_measurements(p)
    good = tmp_path / "g.hsm"
    pl.save_measurements(good, np.ones((2, 2, 3)), 8, masks=np.zeros((2, 2, 3), dtype=np.uint8))
    p.write_bytes(good.read_bytes()[:-1])                    # truncated payload
    with pytest.raises(pl.PipelineFileError):
        pl.load_measurements(p)
    c = np.ones((1, 1, 2), dtype=np.complex128) * (1 + 1j)   # a DFT run: imaginary parts
    pl.save_measurements(p, c, 4)
    with pytest.raises(pl.PipelineFileError):
        pl.load_measurements(p)
    with pytest.raises(ValueError):                          # band index >= n
        pl.save_measurements(p, np.ones((1, 1, 2)), 4, masks=np.array([[[1, 4]]], dtype=np.uint8))
    with pytest.raises(pl.PipelineFileError):
        pl.load_mask(tmp_path / "missing.txt")
    (tmp_path / "m.txt").write_text("seed=1\nn=3\n")
    with pytest.raises(pl.PipelineFileError):
        pl.load_mask(tmp_path / "m.txt")


def _rows():
    out = []
    for r in _inputs()["rows"]:
        r = dict(r)
        r["psnr_db"] = math.inf if r["psnr_db"] == "inf" else r["psnr_db"]
        out.append(pl.SummaryRow(**r))
    return out


def test_report_bytes_match_reference(tmp_path):
    pl.write_report(_rows(), tmp_path / "report.csv")
    assert (tmp_path / "report.csv").read_bytes() == (GOLD / "ref_report.csv").read_bytes()


def test_report_round_trip_and_validation(tmp_path):
    rows = pl.read_report(GOLD / "ref_report.csv")
    assert [r.algorithm for r in rows] == ["cosamp", "admm", "fista", "gomp"]
    assert math.isinf(rows[1].psnr_db) and rows[0].total_iterations == 159000
    with pytest.raises(ValueError):
        pl.SummaryRow("d", "lasso", "λ=1", 1.0, 1, 50.0, 0.1)
    with pytest.raises(ValueError):
        pl.SummaryRow("d", "fista", "λ=1", 1.0, 1, 101.0, 0.1)
    with pytest.raises(ValueError):
        pl.SummaryRow("d", "fista", "λ=1", float("nan"), 1, 50.0, 0.1)
    (tmp_path / "x.csv").write_text("a,b\n")
    with pytest.raises(ValueError):
        pl.read_report(tmp_path / "x.csv")


def test_labels_and_summarize_gate():
    assert pl.param_label("fista", SolverConfig(lam=0.1)) == "λ=0.1"
    assert pl.param_label("cosamp", SolverConfig(kappa=33)) == "κ=33"
    assert pl.tag_of("admm", SolverConfig(lam=100.0)) == "admm_lambda100"
    assert pl.tag_of("gomp", SolverConfig(kappa=27)) == "gomp_kappa27"

    class St:
        n_converged, total_iterations, n_zero_pixels, convergence_pct, recovery_time_s = 5, 0, 2, 100.0, 0.1
    with pytest.raises(ValueError):
        pl.summarize("d", "gomp", SolverConfig(kappa=5), St(), 30.0)
    St.n_zero_pixels = 5
    row = pl.summarize("d", "gomp", SolverConfig(kappa=5), St(), 30.0)
    assert row.param_label == "κ=5" and row.total_iterations == 0


def test_cli_config_errors_exit_2(tmp_path, capsys):
    assert pl.main(["recover", "--input", str(tmp_path), "--algorithm", "lasso"]) == pl.EXIT_CONFIG
    assert pl.main(["recover", "--input", str(tmp_path), "--algorithm", "gomp", "--kappa", "0"]) == pl.EXIT_CONFIG
    # missing run directory contents: I/O error
    assert pl.main(["report", "--input", str(tmp_path)]) == pl.EXIT_IO
