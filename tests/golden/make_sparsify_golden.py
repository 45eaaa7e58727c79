"""Golden fixture for the input-side step FROM THE REFERENCE ITSELF.

Run in the build container (the reference is importable there, not on the GPU
box):  python tests/golden/make_sparsify_golden.py

Calls the unmodified `hypercs.transform.sparsify` (transform.py:73-97) on
seeded real coefficient vectors (the DCT basis is real, so the GPU path sees
real coefficients) for several threshold factors and stores inputs, kept
vectors and the recorded statistics in sparsify.npz.  Vector families: dense
Gaussian, sparse Gaussian (the "never grows the support" family of
test_transform.py:117-122), heavy-tailed, and constant-magnitude vectors with
exactly representable sums (std 0: nothing is zeroed, test_transform.py:110-115).
"""

import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, "/root/reference/pkg/src")

from hypercs.transform import sparsify  # noqa: E402  (the reference package, read-only)


def main():
    rng = np.random.default_rng(2024)
    xs, factors, outs, means, stds, zfs = [], [], [], [], [], []
    n = 224
    families = []
    for _ in range(24):
        families.append(rng.standard_normal(n))
    for _ in range(24):
        families.append(rng.standard_normal(n) * (rng.uniform(size=n) > 0.4))
    for _ in range(12):
        families.append(rng.standard_cauchy(n) * 0.01)
    for v in (2.0, 0.5, 0.25):
        families.append(v * rng.choice([-1.0, 1.0], n))
    for x in families:
        for f in (0.0, 0.1, 0.5, 1.0, 2.0):
            out, st = sparsify(x, f)
            assert np.all(np.imag(out) == 0)
            xs.append(x)
            factors.append(f)
            outs.append(np.real(out).astype(np.float64))
            means.append(st.mean_magnitude)
            stds.append(st.std_magnitude)
            zfs.append(st.zero_fraction)
    np.savez_compressed(HERE / "sparsify.npz", x=np.array(xs), factor=np.array(factors), out=np.array(outs),
                        mean=np.array(means), std=np.array(stds), zero_fraction=np.array(zfs))
    print(f"wrote {len(xs)} sparsify cases")


if __name__ == "__main__":
    main()
