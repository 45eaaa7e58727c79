"""Golden files for the run-directory formats FROM THE REFERENCE ITSELF.

Run in the build container (the reference is importable there, not on the GPU
box):  python tests/golden/make_format_golden.py

Writes, with the unmodified reference writers,
  formats/ref_measurements.hsm  cli.save_measurements (cli.py:68-76), HSM1, a
                                3 x 2 x 5 real-valued complex128 payload, n = 12
  formats/ref_mask.txt          transform.save_mask (transform.py:139-147)
  formats/ref_report.csv        metrics.write_report (metrics.py:123-141) of
                                four SummaryRows (one with an infinite PSNR)
plus formats/inputs.json with the values they were written from, so
tests/test_pipeline.py can check that paper_2401_14762_b200.pipeline reads
these files and writes byte-identical ones.
"""

import json
import math
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent / "formats"
sys.path.insert(0, "/root/reference/pkg/src")

from hypercs.cli import save_measurements  # noqa: E402  (the reference package, read-only)
from hypercs.metrics import SummaryRow, write_report  # noqa: E402
from hypercs.transform import SelectionMask, save_mask  # noqa: E402


def main():
    HERE.mkdir(parents=True, exist_ok=True)
    rng = np.random.default_rng(5)
    meas = rng.standard_normal((3, 2, 5))
    save_measurements(HERE / "ref_measurements.hsm", meas.astype(np.complex128), 12)
    idx = [0, 2, 3, 7, 11]
    save_mask(SelectionMask(n=12, indices=np.array(idx), seed=42), HERE / "ref_mask.txt")
    rows = [
        dict(dataset="salinas", algorithm="gomp", param_label="κ=27", psnr_db=59.8477105, total_iterations=3756956,
             convergence_pct=100.0, recovery_time_s=0.336),
        dict(dataset="jasper", algorithm="fista", param_label="λ=0.1", psnr_db=28.36431, total_iterations=733100,
             convergence_pct=99.987, recovery_time_s=0.0123456789),
        dict(dataset="jasper", algorithm="admm", param_label="λ=100", psnr_db=math.inf, total_iterations=0,
             convergence_pct=100.0, recovery_time_s=1e-6),
        dict(dataset="china", algorithm="cosamp", param_label="κ=33", psnr_db=15.49234, total_iterations=159000,
             convergence_pct=40.5, recovery_time_s=2.5),
    ]
    write_report([SummaryRow(**r) for r in rows], HERE / "ref_report.csv")
    inputs = dict(measurements=meas.tolist(), n=12, mask=dict(n=12, seed=42, indices=idx),
                  rows=[dict(r, psnr_db="inf" if math.isinf(r["psnr_db"]) else r["psnr_db"]) for r in rows])
    (HERE / "inputs.json").write_text(json.dumps(inputs, indent=1, ensure_ascii=False) + "\n")
    print(f"wrote {sorted(p.name for p in HERE.iterdir())}")


if __name__ == "__main__":
    main()
