"""Input side on the GPU: synthetic spectra, sparsify, measure.

Checked against the host generator (synth.generate, numpy) and the reference's
own sparsify (tests/golden/sparsify.npz, made by tests/golden/make_sparsify_golden.py
from hypercs.transform.sparsify, transform.py:73-97), plus the known answers of
the reference's test_transform.py:91-129 restated for real vectors.
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import cpu_solvers as oc  # noqa: E402
from paper_2401_14762_b200 import sparsify as sp  # noqa: E402
from paper_2401_14762_b200 import synth  # noqa: E402

pytestmark = pytest.mark.gpu


def _identity_sparsify(x, factor):
    """GPU sparsify of coefficient vectors: the identity basis makes the two
    GEMMs exact, so the kernel's threshold is the only operation."""
    x = np.atleast_2d(np.asarray(x, dtype=np.float64))
    n = x.shape[1]
    masks = np.tile(np.arange(n, dtype=np.uint8), (x.shape[0], 1))
    out = sp.sparsify_measure(x, np.eye(n), n, rule="meanstd", factor=factor, masks=masks)
    return out


def test_synth_spectra_matches_host_recipe():
    n, P = 224, 3000
    cen, wid, amp, noise, _ = synth._draw(P, n, 5)
    f = sp.synth_spectra(cen, wid, amp, noise).cpu().numpy()
    bands = np.arange(n, dtype=np.float64)
    z = (bands[None, None, :] - cen[:, :, None]) / wid[:, :, None]
    ref = np.clip((amp[:, :, None] * np.exp(-0.5 * z * z)).sum(axis=1) + noise, 0.0, 1.0)
    # exp() may differ from numpy's by an ulp; values are <= 1
    assert np.max(np.abs(f - ref)) <= 4e-16
    assert np.mean(f == ref) > 0.9          # measured: 95% bit-identical


@pytest.mark.parametrize("name,x_range", [("jasper", None), ("china", (0, 60)), ("scaling", (508, 516))])
def test_generate_device_matches_host_generator(name, x_range):
    host = synth.generate_named(name, x_range=x_range)
    dev = synth.generate_named_device(name, x_range=x_range, with_coeffs=True)
    assert dev.seeds == host.seeds and dev.shape == host.shape
    assert np.array_equal(dev.masks.cpu().numpy(), host.masks)          # integer work: bit-exact
    c = dev.coeffs.cpu().numpy()
    scale = np.abs(host.coeffs).max(axis=1, keepdims=True)
    # identical threshold decisions except coefficients within rounding of T max|c|
    thr = synth.SPARSIFY_T * scale
    near = np.abs(np.abs(host.coeffs) - thr) <= 1e-12 * scale
    flips = ((c == 0) != (host.coeffs == 0)) & ~near
    assert not flips.any(), f"{int(flips.sum())} threshold decisions differ away from the threshold"
    assert int(((c == 0) != (host.coeffs == 0)).sum()) <= max(1, host.coeffs.size // 10 ** 6)
    ok = ~((c == 0) != (host.coeffs == 0)).any(axis=1)
    assert np.max(np.abs(c - host.coeffs)[ok]) <= 1e-13
    assert np.max(np.abs(dev.spectra.cpu().numpy() - host.spectra)[ok]) <= 1e-13
    assert np.max(np.abs(dev.y.cpu().numpy() - host.y)[ok]) <= 1e-13
    assert abs(dev.zero_fraction - float(np.mean(host.coeffs == 0))) <= 1e-6


def test_sparsify_matches_reference_golden(golden_dir):
    z = np.load(golden_dir / "sparsify.npz")
    x, fac, out = z["x"], z["factor"], z["out"]
    for f in np.unique(fac):
        sel = fac == f
        got = _identity_sparsify(x[sel], float(f))
        kept = got.coeffs.cpu().numpy()
        # GPU mean/std sum in another order: decisions may differ only where
        # (|x| - mean) is within rounding of factor * std
        mags = np.abs(x[sel])
        slack = np.abs((mags - z["mean"][sel][:, None]) - f * z["std"][sel][:, None])
        differ = (kept != out[sel])
        assert not (differ & (slack > 1e-12)).any()
        assert np.array_equal(kept[~differ], out[sel][~differ])
        # kept entries are bit-identical to the input (transform.py:95-96)
        nz = kept != 0
        assert np.array_equal(kept[nz], x[sel][nz])
        assert np.array_equal(got.y.cpu().numpy(), kept)       # identity basis, all bands measured


def test_sparsify_known_answers():                 # test_transform.py:91-129, real vectors
    got = _identity_sparsify([4.0, -1.0, 1.0, 2.0], 0.1)
    assert got.coeffs.cpu().numpy().tolist() == [[4.0, 0.0, 0.0, 0.0]]
    assert got.zero_fraction == pytest.approx(0.75)
    got = _identity_sparsify([4.0, -1.0, 1.0, 2.0], 0.0)
    assert got.coeffs.cpu().numpy().tolist() == [[4.0, 0.0, 0.0, 2.0]]
    x = np.array([0.1, 7.123456789012345e-1 * 9, 1e-3])
    k = _identity_sparsify(x, 0.0).coeffs.cpu().numpy()[0]
    assert np.array_equal(k[k != 0], x[k != 0])
    x = np.array([5.0, -5.0, 5.0])
    got = _identity_sparsify(x, 3.0)
    assert np.array_equal(got.coeffs.cpu().numpy()[0], x) and got.zeroed == 0
    rng = np.random.default_rng(3)
    for _ in range(20):
        x = rng.standard_normal(40) * (rng.uniform(size=40) > 0.4)
        k = _identity_sparsify(x, rng.uniform(0.0, 2.0)).coeffs.cpu().numpy()[0]
        assert np.count_nonzero(k) <= np.count_nonzero(x)
    with pytest.raises(ValueError):
        _identity_sparsify([1.0], -0.5)


def test_meanstd_rule_in_the_dct_domain_matches_oracle():
    cube = synth.generate(20, 50, 198, seed=3)
    got = sp.sparsify_measure(cube.spectra, cube.basis, cube.m, rule="meanstd", factor=0.5, masks=cube.masks)
    c, fs, y = oc.sparsify_measure(cube.spectra, cube.basis, cube.masks, rule="meanstd", factor=0.5)
    gc = got.coeffs.cpu().numpy()
    assert np.mean((gc == 0) == (c == 0)) > 0.9999
    ok = ((gc == 0) == (c == 0)).all(axis=1)
    assert np.max(np.abs(gc - c)[ok]) <= 1e-13
    assert np.max(np.abs(got.y.cpu().numpy() - y)[ok]) <= 1e-13
    assert np.max(np.abs(got.spectra.cpu().numpy() - fs)[ok]) <= 1e-13


def test_masks_from_keys_take_the_smallest_with_ties_to_the_lower_index():
    n, m = 37, 9
    rng = np.random.default_rng(1)
    keys = rng.random((64, n))
    keys[0, :] = 0.5                                     # all tied: the first m bands
    keys[1, ::2] = -1.0                                  # negatives order below positives
    keys[2, 5] = 0.0
    keys[2, 6] = -0.0
    f = rng.random((64, n))
    got = sp.sparsify_measure(f, np.eye(n), m, rule="maxrel", factor=0.0, keys=keys)
    mk = got.masks.cpu().numpy().astype(np.int64)
    exp = np.sort(np.argsort(keys, axis=1, kind="stable")[:, :m], axis=1)
    assert np.array_equal(mk[3:], exp[3:])
    assert mk[0].tolist() == list(range(m))
    assert mk[1].tolist() == list(range(0, n, 2))[:m]
    assert 5 in mk[2] and 6 in mk[2]
    assert np.array_equal(got.y.cpu().numpy(), np.take_along_axis(f, mk, axis=1))


def test_empty_and_invalid_inputs():
    b = synth.dct_basis(16)
    got = sp.sparsify_measure(np.zeros((0, 16)), b, 6, rule="maxrel", factor=0.1, masks=np.zeros((0, 6), np.uint8))
    assert got.y.shape == (0, 6) and got.zeroed == 0
    with pytest.raises(ValueError):
        sp.sparsify_measure(np.zeros((2, 16)), b, 17, masks=np.zeros((2, 17), np.uint8))
    with pytest.raises(ValueError):
        sp.sparsify_measure(np.zeros((2, 16)), b, 6, rule="median", masks=np.zeros((2, 6), np.uint8))
    with pytest.raises(ValueError):
        sp.sparsify_measure(np.zeros((2, 16)), b, 6)


@pytest.mark.parametrize("P,n,offset", [(5000, 224, 0), (777, 198, 0), (333, 154, 1), (1, 1, 0)])
def test_sse_coeff_partials_parseval(P, n, offset):
    """Coefficient-domain SSE equals the spectral-domain SSE
    of the reference's psnr (metrics.py:30-55) for the orthonormal DCT-II basis:
    ||f_ref - Psi x||^2 = ||c_ref - x||^2.  offset=1 exercises the unaligned
    (scalar) path; n*P odd exercises the double2 tail."""
    from paper_2401_14762_b200.metrics import psnr_partials, sse_coeff_partials
    rng = np.random.default_rng(P + n)
    basis = synth.dct_basis(n)
    c = rng.standard_normal((P, n)) * (rng.random((P, n)) < 0.1)
    x = c + 1e-3 * rng.standard_normal((P, n))
    f = c @ basis.T                       # f_p = Psi c_p
    dev = torch.device("cuda")
    flat_c = torch.as_tensor(np.concatenate([np.zeros(offset), c.ravel()]), device=dev)[offset:].view(P, n)
    flat_x = torch.as_tensor(np.concatenate([np.zeros(offset), x.ravel()]), device=dev)[offset:].view(P, n)
    got = float(sse_coeff_partials(flat_c, flat_x).item())
    want = float(np.sum((c - x) ** 2))
    assert abs(got - want) <= 1e-12 * want
    spec = psnr_partials(torch.as_tensor(f, device=dev), torch.as_tensor(x, device=dev),
                         torch.as_tensor(basis, device=dev)).cpu().numpy()
    assert abs(got - spec[0]) <= 1e-9 * spec[0]


def test_sse_coeff_partials_rejects_mismatch():
    from paper_2401_14762_b200.metrics import sse_coeff_partials
    a = torch.zeros((4, 8), dtype=torch.float64, device="cuda")
    with pytest.raises(ValueError):
        sse_coeff_partials(a, torch.zeros((4, 9), dtype=torch.float64, device="cuda"))
