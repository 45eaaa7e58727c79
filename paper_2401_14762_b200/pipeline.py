"""Run-directory pipeline around the GPU path.

The reference's CLI chains file-based stages in a run directory
(`cli.py:97-219`, `cli.py:460-505`): sparsify -> compress -> recover -> report.
This module keeps its artefacts and record formats where they carry the
recovery path, and extends them for BASELINE's per-pixel masks:

* measurements: the reference's ``HSM1`` file (`cli.py:53-91`: magic, four
  little-endian uint32 x/y/m/n, complex128 payload) is read and written
  unchanged for a shared mask.  ``HSM2`` adds per-pixel masks: magic, five
  uint32 x/y/m/n/flags, float64 measurements (the reference's imaginary parts
  are identically 0 for a real basis), then, when ``flags & 1``, the (x, y, m)
  uint8 band indices of every pixel (sorted, < n <= 256).
* mask.txt: the reference's ``seed=/n=/indices=`` text (`transform.py:139-165`)
  for a shared mask; a per-pixel run writes ``seed=``, ``n=``, ``m=`` and
  ``indices=per-pixel`` (the indices live in the HSM2 payload).
* recover (`cli.run_recover`, `cli.py:171-219`) routes to ``recover_cube`` on
  the GPU with the DCT-II basis, and writes the reference's
  ``pixels_{tag}.csv`` (same columns) and ``run_{tag}.json`` (same keys); the
  recovered spectra go to ``recovered_{tag}.npy`` (float64 x, y, n) instead of
  the reference's HSC1 cube container (its cube I/O is out of scope).
* report (`cli.run_report`, `metrics.summarize/write_report/read_report`,
  `metrics.py:67-170`): Table-1 rows with the reference's header, comment
  line, ordering and float formatting; PSNR against ``sparsified.npy``.
* synth: a run directory from the frozen synthetic generator (the stand-in
  for the reference's sparsify + compress of a real dataset), input side on
  the GPU.

Exit codes follow `cli.py:46-49`: 0 ok, 2 configuration error, 3 I/O or
file-format error, 4 completed with numerically failed pixels.
"""

import argparse
import csv
import json
import math
import struct
import sys
from dataclasses import asdict, dataclass
from pathlib import Path

import numpy as np

from .metrics import UndefinedMetricError
from .solvers import CONVEX_SOLVERS, SOLVERS, SolverConfig, recover_cube

EXIT_OK, EXIT_CONFIG, EXIT_IO, EXIT_PARTIAL = 0, 2, 3, 4

MEAS_MAGIC = b"HSM1"
MEAS_HEADER = struct.Struct("<IIII")
MEAS_MAGIC_PP = b"HSM2"
MEAS_HEADER_PP = struct.Struct("<IIIII")
FLAG_PER_PIXEL = 1

SPARSIFIED_FILE = "sparsified.npy"
SPARSIFY_STATS_FILE = "sparsify_stats.json"
MEASUREMENTS_FILE = "measurements.hsm"
MASK_FILE = "mask.txt"
REPORT_FILE = "report.csv"

REPORT_COMMENT = "# recovery_time_s is wall-clock and varies between runs"
REPORT_HEADER = ("dataset", "algorithm", "param", "psnr_db", "iterations", "convergence_pct", "recovery_time_s")
IDENTICAL = "identical"


class ConfigError(Exception):
    """Bad or missing run parameters (exit code 2)."""


class PipelineFileError(Exception):
    """A pipeline artefact is missing pieces or does not parse (exit code 3)."""


# ------------------------------------------------------------------ measurement files


def save_measurements(path, measurements, n, masks=None):
    """Write HSM1 (shared mask: ``masks`` None, the reference's complex128
    layout) or HSM2 (``masks`` (x, y, m) uint8 per-pixel band indices, real
    float64 payload)."""
    meas = np.asarray(measurements)
    if meas.ndim != 3:
        raise ValueError("measurements must be (x, y, m)")
    x, y, m = meas.shape
    with open(path, "wb") as fh:
        if masks is None:
            fh.write(MEAS_MAGIC)
            fh.write(MEAS_HEADER.pack(x, y, m, n))
            fh.write(np.ascontiguousarray(meas, dtype=np.complex128).tobytes())
            return
        masks = np.asarray(masks)
        if masks.shape != meas.shape:
            raise ValueError("per-pixel masks must have the measurements' (x, y, m) shape")
        if n > 256 or (masks.size and int(masks.max()) >= n):
            raise ValueError("band indices must be < n <= 256")
        if np.iscomplexobj(meas):
            if np.any(meas.imag != 0):
                raise ValueError("HSM2 stores real measurements; imaginary parts must be 0")
            meas = meas.real
        fh.write(MEAS_MAGIC_PP)
        fh.write(MEAS_HEADER_PP.pack(x, y, m, n, FLAG_PER_PIXEL))
        fh.write(np.ascontiguousarray(meas, dtype=np.float64).tobytes())
        fh.write(np.ascontiguousarray(masks, dtype=np.uint8).tobytes())


def load_measurements(path):
    """Read HSM1 or HSM2.  Returns (measurements float64 (x, y, m), n, masks
    (x, y, m) uint8 or None).  HSM1's complex payload must be real (a real
    basis gives imaginary parts of exactly 0)."""
    path = Path(path)
    try:
        raw = path.read_bytes()
    except OSError as exc:
        raise PipelineFileError(f"{path}: {exc}") from None
    if raw[:4] == MEAS_MAGIC and len(raw) >= 4 + MEAS_HEADER.size:
        x, y, m, n = MEAS_HEADER.unpack_from(raw, 4)
        payload = raw[4 + MEAS_HEADER.size:]
        if len(payload) != x * y * m * 16:
            raise PipelineFileError(f"{path}: payload size does not match the header")
        meas = np.frombuffer(payload, dtype=np.complex128).reshape(x, y, m)
        if np.any(meas.imag != 0):
            raise PipelineFileError(f"{path}: complex measurements (a DFT run) are not supported by the "
                                    "real-FP64 GPU path")
        return np.ascontiguousarray(meas.real), n, None
    if raw[:4] == MEAS_MAGIC_PP and len(raw) >= 4 + MEAS_HEADER_PP.size:
        x, y, m, n, flags = MEAS_HEADER_PP.unpack_from(raw, 4)
        payload = raw[4 + MEAS_HEADER_PP.size:]
        count = x * y * m
        want = count * 8 + (count if flags & FLAG_PER_PIXEL else 0)
        if len(payload) != want:
            raise PipelineFileError(f"{path}: payload size does not match the header")
        meas = np.frombuffer(payload[:count * 8], dtype=np.float64).reshape(x, y, m).copy()
        masks = None
        if flags & FLAG_PER_PIXEL:
            masks = np.frombuffer(payload[count * 8:], dtype=np.uint8).reshape(x, y, m).copy()
            if masks.size and int(masks.max()) >= n:
                raise PipelineFileError(f"{path}: band index outside [0, n)")
        return meas, n, masks
    raise PipelineFileError(f"{path}: not a measurement file")


# ------------------------------------------------------------------ mask files


def save_mask(path, n, seed, indices=None, m=None):
    """The reference's mask text (shared ``indices``) or the per-pixel marker."""
    lines = [f"seed={int(seed)}", f"n={int(n)}"]
    if indices is None:
        if m is None:
            raise ValueError("a per-pixel mask file needs m")
        lines += [f"m={int(m)}", "indices=per-pixel"]
    else:
        lines.append("indices=" + ",".join(str(int(i)) for i in indices))
    Path(path).write_text("\n".join(lines) + "\n", encoding="ascii")


def load_mask(path):
    """dict(seed, n, m, indices: ndarray or None for per-pixel)."""
    fields = {}
    try:
        text = Path(path).read_text(encoding="ascii")
    except (OSError, UnicodeDecodeError) as exc:
        raise PipelineFileError(f"{path}: {exc}") from None
    for line in text.splitlines():
        line = line.strip()
        if line:
            key, _, value = line.partition("=")
            fields[key.strip()] = value.strip()
    try:
        seed, n = int(fields["seed"]), int(fields["n"])
        if fields["indices"] == "per-pixel":
            return dict(seed=seed, n=n, m=int(fields["m"]), indices=None)
        idx = np.array([int(t) for t in fields["indices"].split(",")], dtype=np.intp)
    except (KeyError, ValueError) as exc:
        raise PipelineFileError(f"unreadable mask file {path}: {exc}") from None
    return dict(seed=seed, n=n, m=len(idx), indices=idx)


# ------------------------------------------------------------------ report rows


@dataclass
class SummaryRow:
    """One benchmark line: dataset x algorithm x parameter (metrics.py:67-86)."""

    dataset: str
    algorithm: str
    param_label: str
    psnr_db: float
    total_iterations: int
    convergence_pct: float
    recovery_time_s: float

    def __post_init__(self):
        if self.algorithm not in SOLVERS:
            raise ValueError(f"unknown algorithm {self.algorithm!r}")
        if not 0.0 <= self.convergence_pct <= 100.0:
            raise ValueError("convergence_pct outside [0, 100]")
        if math.isnan(self.psnr_db):
            raise ValueError("psnr_db is NaN")


def param_label(algorithm, config):
    """lambda for the convex solvers, kappa for the greedy ones (metrics.py:89-94)."""
    return f"λ={config.lam:g}" if algorithm in CONVEX_SOLVERS else f"κ={config.kappa}"


def tag_of(algorithm, config):
    return f"{algorithm}_lambda{config.lam:g}" if algorithm in CONVEX_SOLVERS else f"{algorithm}_kappa{config.kappa}"


def summarize(dataset, algorithm, config, stats, psnr_db):
    """One recovery folded into a SummaryRow, with the reference's sanity gate
    (metrics.py:97-116)."""
    if stats.n_converged > 0 and stats.total_iterations == 0 and stats.n_converged > stats.n_zero_pixels:
        raise ValueError("impossible aggregate: converged pixels but no iterations")
    return SummaryRow(dataset=dataset, algorithm=algorithm, param_label=param_label(algorithm, config),
                      psnr_db=psnr_db, total_iterations=stats.total_iterations,
                      convergence_pct=stats.convergence_pct, recovery_time_s=stats.recovery_time_s)


def write_report(rows, path):
    """Deterministic CSV (metrics.py:123-141): sorted rows, fixed formats."""
    ordered = sorted(rows, key=lambda r: (r.dataset, r.algorithm, r.param_label))
    with open(path, "w", newline="", encoding="utf-8") as fh:
        fh.write(REPORT_COMMENT + "\n")
        w = csv.writer(fh, lineterminator="\n")
        w.writerow(REPORT_HEADER)
        for r in ordered:
            w.writerow([r.dataset, r.algorithm, r.param_label,
                        IDENTICAL if math.isinf(r.psnr_db) else f"{r.psnr_db:.4f}",
                        r.total_iterations, f"{r.convergence_pct:.2f}", f"{r.recovery_time_s:.6f}"])


def read_report(path):
    """Parse write_report output back into SummaryRows (metrics.py:144-170)."""
    with open(path, newline="", encoding="utf-8") as fh:
        lines = [ln for ln in fh if not ln.startswith("#")]
    reader = csv.reader(lines)
    header = next(reader, None)
    if header is None or tuple(header) != REPORT_HEADER:
        raise ValueError(f"{path}: not a report file")
    rows = []
    for rec in reader:
        if rec:
            ds, algo, param, ps, it, conv, el = rec
            rows.append(SummaryRow(ds, algo, param, math.inf if ps == IDENTICAL else float(ps), int(it),
                                   float(conv), float(el)))
    return rows


def _psnr_abs_max(reference, reconstruction):
    peak = float(np.max(np.abs(reference)))
    if peak <= 0:
        raise UndefinedMetricError(f"non-positive peak {peak} under 'abs-max'")
    d = reference - reconstruction
    mse = float(np.vdot(d, d).real) / d.size
    return math.inf if mse == 0.0 else 10.0 * math.log10(peak * peak / mse)


# ------------------------------------------------------------------ stages


def run_synth(out_dir, cube="jasper", seed=0, x_range=None, dataset=None):
    """A run directory from the frozen generator (synth.py v1), input side on
    the GPU: sparsified.npy (reference spectra), measurements.hsm (HSM2,
    per-pixel masks), mask.txt, sparsify_stats.json."""
    from . import synth
    spec = synth.CUBES[cube]
    c = synth.generate_named_device(cube, seed=seed, x_range=x_range)
    rows, ydim = c.shape
    n, m = c.n, c.m
    out_dir = Path(out_dir)
    out_dir.mkdir(parents=True, exist_ok=True)
    np.save(out_dir / SPARSIFIED_FILE, c.spectra.cpu().numpy().reshape(rows, ydim, n))
    save_measurements(out_dir / MEASUREMENTS_FILE, c.y.cpu().numpy().reshape(rows, ydim, m), n,
                      masks=c.masks.cpu().numpy().reshape(rows, ydim, m))
    save_mask(out_dir / MASK_FILE, n, seed, m=m)
    stats = {"dataset": dataset or f"synthetic-{cube}", "threshold_factor": synth.SPARSIFY_T,
             "zero_fraction": c.zero_fraction, "x": rows, "y": ydim, "bands": n,
             "generator": synth.GENERATOR_VERSION,
             "seeds": list(c.seeds), "shape_of": spec}
    (out_dir / SPARSIFY_STATS_FILE).write_text(json.dumps(stats, indent=1) + "\n")
    print(f"[synth] {out_dir}: {rows}x{ydim}x{n}, m={m} per-pixel, zero_fraction={c.zero_fraction:.4f}")
    return stats


def _write_pixel_log(path, stats, y_dim):
    """The reference's per-pixel CSV (cli.py:148-168), from the per-pixel arrays."""
    with open(path, "w", newline="", encoding="utf-8") as fh:
        w = csv.writer(fh, lineterminator="\n")
        w.writerow(["x", "y", "iterations", "converged", "elapsed_s", "final_delta", "failed"])
        for index in range(stats.n_pixels):
            ix, iy = divmod(index, y_dim)
            fa = int(stats.failed_at[index])
            if fa >= 0:
                w.writerow([ix, iy, fa, 0, "", "", 1])
            else:
                w.writerow([ix, iy, int(stats.iterations[index]), int(stats.converged[index]),
                            f"{float(stats.elapsed[index]):.6f}", f"{float(stats.final_delta[index]):.3e}", 0])


def run_recover(run_dir, algorithm, config, jobs=1, dataset=None):
    """cli.run_recover (cli.py:171-219) on the GPU: per-pixel or shared
    dictionary from the run's mask, DCT-II basis, spectra = Psi x."""
    from .transform import Dictionary, SelectionMask, build_dct_basis, build_dictionary
    run_dir = Path(run_dir)
    meas, n, masks = load_measurements(run_dir / MEASUREMENTS_FILE)
    mk = load_mask(run_dir / MASK_FILE)
    if mk["n"] != n or mk["m"] != meas.shape[2]:
        raise PipelineFileError(f"{run_dir}: mask does not match the measurement file")
    if (mk["indices"] is None) != (masks is not None):
        raise PipelineFileError(f"{run_dir}: mask.txt and the measurement file disagree on per-pixel masks")
    if dataset is None:
        sp = run_dir / SPARSIFY_STATS_FILE
        if sp.exists():
            dataset = json.loads(sp.read_text()).get("dataset")
        dataset = dataset or run_dir.name
    basis = build_dct_basis(n)
    if masks is not None:
        dic = Dictionary.per_pixel(basis, masks)
    else:
        dic = build_dictionary(basis, SelectionMask(n=n, indices=mk["indices"], seed=mk["seed"]))
    cube, stats = recover_cube(meas, dic, config, algorithm, jobs)
    x_dim, y_dim = meas.shape[:2]
    spectra = (np.asarray(cube).reshape(-1, n) @ basis.matrix.T).reshape(x_dim, y_dim, n)
    tag = tag_of(algorithm, config)
    np.save(run_dir / f"recovered_{tag}.npy", spectra)
    _write_pixel_log(run_dir / f"pixels_{tag}.csv", stats, y_dim)
    meta = {
        "dataset": dataset, "algorithm": algorithm, "param_label": param_label(algorithm, config), "tag": tag,
        "n_pixels": stats.n_pixels, "n_converged": stats.n_converged, "n_failed": stats.n_failed,
        "n_zero_pixels": stats.n_zero_pixels, "total_iterations": stats.total_iterations,
        "mean_iterations_per_pixel": stats.total_iterations / stats.n_pixels,
        "convergence_pct": stats.convergence_pct, "recovery_time_s": stats.recovery_time_s,
        "recovered_file": f"recovered_{tag}.npy", "pixels_file": f"pixels_{tag}.csv",
        "config": asdict(config), "backend": "b200 (libhypercs_b200.so)",
    }
    (run_dir / f"run_{tag}.json").write_text(json.dumps(meta, indent=1, default=str) + "\n")
    print(f"[recover] {tag}: {stats.n_converged}/{stats.n_pixels} converged, "
          f"{stats.total_iterations} iterations, {stats.n_failed} failed")
    return stats, tag


def run_report(run_dir, out_path=None, dataset=None):
    """cli.run_report (cli.py:222-262): one row per run_*.json, PSNR of the
    recovered spectra against sparsified.npy (abs-max peak)."""
    run_dir = Path(run_dir)
    try:
        ref = np.load(run_dir / SPARSIFIED_FILE)
    except OSError as exc:
        raise PipelineFileError(f"{run_dir}: {exc}") from None
    rows = []
    for mp in sorted(run_dir.glob("run_*.json")):
        try:
            meta = json.loads(mp.read_text())
            f = {k: meta[k] for k in ("algorithm", "param_label", "total_iterations", "convergence_pct",
                                      "recovery_time_s", "n_converged", "n_zero_pixels", "recovered_file")}
            f["dataset"] = dataset or meta["dataset"]
        except (KeyError, json.JSONDecodeError) as exc:
            raise PipelineFileError(f"{mp}: unreadable recovery record: {exc}") from None
        if f["n_converged"] > 0 and f["total_iterations"] == 0 and f["n_converged"] > f["n_zero_pixels"]:
            raise PipelineFileError(f"{mp}: converged pixels with zero iterations")
        try:
            rec = np.load(run_dir / f["recovered_file"])
        except OSError as exc:
            raise PipelineFileError(f"{mp}: {exc}") from None
        rows.append(SummaryRow(f["dataset"], f["algorithm"], f["param_label"], _psnr_abs_max(ref, rec),
                               f["total_iterations"], f["convergence_pct"], f["recovery_time_s"]))
    if not rows:
        raise PipelineFileError(f"{run_dir}: no recovery records to report")
    out_path = out_path or run_dir / REPORT_FILE
    write_report(rows, out_path)
    print(f"[report] {out_path}: {len(rows)} rows")
    return rows


# ------------------------------------------------------------------ command line


def _configs(args):
    algos = [a.strip() for a in args.algorithm.split(",") if a.strip()]
    out = []
    for algo in algos:
        if algo not in SOLVERS:
            raise ConfigError(f"unknown algorithm {algo!r}")
        common = dict(epsilon=args.epsilon, max_iter=args.max_iter, time_limit=None)
        if algo in CONVEX_SOLVERS:
            for lam in args.lam:
                out.append((algo, SolverConfig(lam=lam, alpha=args.alpha, **common)))
        else:
            for kappa in args.kappa:
                extra = dict(atoms_per_iter=args.atoms_per_iter) if args.atoms_per_iter else {}
                out.append((algo, SolverConfig(kappa=kappa, mu=args.mu, **extra, **common)))
    return out


def build_parser():
    ap = argparse.ArgumentParser(prog="python -m paper_2401_14762_b200",
                                 description="GPU recovery stages over a run directory (hypercs cli.py layout)")
    sub = ap.add_subparsers(dest="cmd", required=True)
    s = sub.add_parser("synth", help="synthetic run directory (input side on the GPU)")
    s.add_argument("--out", required=True)
    s.add_argument("--cube", default="jasper")
    s.add_argument("--seed", type=int, default=0)
    s.add_argument("--rows", type=int, default=None, help="first ROWS x-rows only")
    s.add_argument("--dataset")
    for name in ("recover", "bench"):
        r = sub.add_parser(name)
        r.add_argument("--input", required=(name == "recover"), help="run directory")
        if name == "bench":
            r.add_argument("--out", required=True)
            r.add_argument("--cube", default="jasper")
            r.add_argument("--seed", type=int, default=0)
            r.add_argument("--rows", type=int, default=None)
        r.add_argument("--algorithm", required=True, help="comma-separated: fista,admm,gomp,biht,cosamp")
        r.add_argument("--lam", type=float, nargs="+", default=[0.1])
        r.add_argument("--kappa", type=int, nargs="+", default=[10])
        r.add_argument("--atoms-per-iter", dest="atoms_per_iter", type=int, default=None)
        r.add_argument("--mu", type=float, default=0.1)
        r.add_argument("--alpha", type=float, default=1.8)
        r.add_argument("--epsilon", type=float, default=1e-8)
        r.add_argument("--max-iter", dest="max_iter", type=int, default=None)
        r.add_argument("--jobs", type=int, default=1)
        r.add_argument("--dataset")
    p = sub.add_parser("report")
    p.add_argument("--input", required=True)
    p.add_argument("--out")
    p.add_argument("--dataset")
    return ap


def main(argv=None):
    args = build_parser().parse_args(argv)
    try:
        if args.cmd == "synth":
            run_synth(args.out, args.cube, args.seed, (0, args.rows) if args.rows else None, args.dataset)
            return EXIT_OK
        if args.cmd == "report":
            run_report(args.input, args.out, args.dataset)
            return EXIT_OK
        configs = _configs(args)
        run_dir = args.input
        if args.cmd == "bench":
            run_dir = args.out
            run_synth(run_dir, args.cube, args.seed, (0, args.rows) if args.rows else None, args.dataset)
        failed = 0
        for algo, cfg in configs:
            stats, _ = run_recover(run_dir, algo, cfg, args.jobs, args.dataset)
            failed += stats.n_failed
        if args.cmd == "bench":
            run_report(run_dir, None, args.dataset)
        return EXIT_PARTIAL if failed else EXIT_OK
    except (ConfigError, ValueError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return EXIT_CONFIG
    except (PipelineFileError, OSError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return EXIT_IO


if __name__ == "__main__":
    sys.exit(main())
