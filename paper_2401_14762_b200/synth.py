"""Frozen synthetic hyperspectral cubes for the BASELINE.json configs.

The reference's datasets (Jasper Ridge, China, Salinas; `PAPER.md:35,69,106`)
are not available here, so seeded synthetic cubes of the same shapes stand in
for them.  The recipe is BASELINE.json's, frozen once (generator version
``GENERATOR_VERSION``); the interpretation choices SURVEY.md §8(d) leaves open
are fixed as follows and recorded in DESIGN.md:

* "width" is the Gaussian sigma: bump = a * exp(-0.5 * ((b - c) / w)**2);
* N(0, 0.01) is additive noise with sigma 0.01;
* per pixel 1..4 bumps, centre U[0, B), width U[5, 40], amplitude U[0.1, 1];
  a pixel always draws 4 bump parameter sets and zeroes the amplitudes of the
  bumps past its count (so the random stream does not depend on the count);
* clip to [0, 1]; coefficients c = C f with C the orthonormal DCT-II; entries
  with |c| < 0.1 * max|c| (per pixel) are zeroed; the reference spectra are
  f_s = Psi c_s with Psi = C^T (synthesis basis);
* per-pixel mask: the M = floor(0.4 B + 0.5) smallest of B uniform keys,
  sorted ascending (same M rule as `transform.py:131`);
* y = f_s[mask];
* the 2048x868 scaling cube tiles the 512x217 generator 4x4; tile (tx, ty)
  uses seed ``base_seed + 4 * tx + ty``.

This is the only place inputs are made; both the oracle and the GPU path
consume the arrays it returns, so parity never depends on these choices.
"""

import math
from dataclasses import dataclass

import numpy as np

GENERATOR_VERSION = "hcs-synth-v1"
SAMPLE_RATIO = 0.4
SPARSIFY_T = 0.1


def dct_basis(n):
    """Orthonormal synthesis basis Psi (n x n): f = Psi @ c, Psi = C^T with
    C the orthonormal DCT-II, C[k, j] = s_k cos(pi k (2 j + 1) / (2 n)).

    Built in closed form on the host in FP64; the same array is handed to the
    oracle and to the GPU so basis rounding is identical on both sides.
    """
    if n < 1:
        raise ValueError("basis size must be >= 1")
    k = np.arange(n, dtype=np.int64)[:, None]
    j = np.arange(n, dtype=np.int64)[None, :]
    # exact integer range reduction of k (2j+1) modulo the period 4n keeps the
    # cosine argument in [0, 2 pi) so the basis is orthonormal to ~1e-16
    q = (k * (2 * j + 1)) % (4 * n)
    # libm cosine over the 4n distinct angles (bit-stable across hosts of one
    # image, unlike SIMD-dispatched np.cos)
    table = np.array([math.cos(math.pi * i / (2.0 * n)) for i in range(4 * n)])
    c = table[q] * math.sqrt(2.0 / n)
    c[0, :] *= 1.0 / math.sqrt(2.0)
    return np.ascontiguousarray(c.T)


def measured_count(n, ratio=SAMPLE_RATIO):
    """round-half-up(ratio * n), the reference's rule (`transform.py:131`)."""
    return int(np.floor(ratio * n + 0.5))


@dataclass
class SyntheticCube:
    """One synthetic measurement problem, pixel-major (x-major raster order).

    basis        (n, n) float64 synthesis matrix Psi
    coeffs       (P, n) float64 sparsified DCT coefficients (ground truth)
    spectra      (P, n) float64 reference spectra f_s = Psi c (PSNR reference)
    masks        (P, m) uint8 sorted measured band indices
    y            (P, m) float64 measurements f_s[mask]
    shape        (x, y) spatial shape, P = x * y
    seeds        seeds used (one per tile)
    """

    basis: np.ndarray
    coeffs: np.ndarray
    spectra: np.ndarray
    masks: np.ndarray
    y: np.ndarray
    shape: tuple
    seeds: tuple
    version: str = GENERATOR_VERSION

    @property
    def n(self):
        return int(self.basis.shape[0])

    @property
    def m(self):
        return int(self.masks.shape[1])

    @property
    def n_pixels(self):
        return int(self.y.shape[0])


def _draw(n_pix, n, seed):
    """The random stream of one seeded tile (the only draws the generator
    makes, in this order): bump centres, widths and count-masked amplitudes
    (n_pix x 4), additive noise and mask keys (n_pix x n)."""
    rng = np.random.default_rng(seed)
    counts = rng.integers(1, 5, size=n_pix)
    centres = rng.uniform(0.0, float(n), size=(n_pix, 4))
    widths = rng.uniform(5.0, 40.0, size=(n_pix, 4))
    amps = rng.uniform(0.1, 1.0, size=(n_pix, 4))
    amps[np.arange(4)[None, :] >= counts[:, None]] = 0.0
    noise = rng.normal(0.0, 0.01, size=(n_pix, n))
    keys = rng.random((n_pix, n))
    return centres, widths, amps, noise, keys


def _tile(n_pix, n, basis, seed, chunk=1 << 16):
    """Spectra, coefficients, masks and measurements for one seeded tile."""
    m = measured_count(n)
    centres, widths, amps, noise, keys = _draw(n_pix, n, seed)

    bands = np.arange(n, dtype=np.float64)
    coeffs = np.empty((n_pix, n))
    spectra = np.empty((n_pix, n))
    for lo in range(0, n_pix, chunk):
        hi = min(n_pix, lo + chunk)
        z = (bands[None, None, :] - centres[lo:hi, :, None]) / widths[lo:hi, :, None]
        f = (amps[lo:hi, :, None] * np.exp(-0.5 * z * z)).sum(axis=1) + noise[lo:hi]
        np.clip(f, 0.0, 1.0, out=f)
        c = f @ basis                      # rows: c_p^T = f_p^T Psi  (c = Psi^T f)
        mag = np.abs(c)
        c[mag < SPARSIFY_T * mag.max(axis=1, keepdims=True)] = 0.0
        coeffs[lo:hi] = c
        spectra[lo:hi] = c @ basis.T       # f_s = Psi c
    masks = np.sort(np.argpartition(keys, m - 1, axis=1)[:, :m], axis=1).astype(np.uint8)
    y = np.take_along_axis(spectra, masks.astype(np.intp), axis=1)
    return coeffs, spectra, masks, np.ascontiguousarray(y)


def _tile_job(args):
    n_pix, n, seed = args
    return _tile(n_pix, n, dct_basis(n), seed)


def generate(x_dim, y_dim, n, seed=0, tiles=(1, 1), x_range=None, workers=1):
    """Synthetic cube of shape (x_dim, y_dim, n), optionally tiled.

    With tiles=(tx, ty) the cube is made of tx*ty independent tiles of size
    (x_dim/tx, y_dim/ty), tile (i, j) seeded with seed + ty*i + j.
    ``x_range=(x0, x1)`` returns only rows x0..x1-1 (a rank's slab; only the
    tiles it touches are generated).  ``workers`` > 1 generates tiles in a
    process pool (results are identical).
    """
    if n > 256:
        raise ValueError("band indices are stored as uint8: n must be <= 256")
    tx, ty = tiles
    if x_dim % tx or y_dim % ty:
        raise ValueError("tiles must divide the cube")
    x0, x1 = x_range if x_range is not None else (0, x_dim)
    if not 0 <= x0 <= x1 <= x_dim:
        raise ValueError("bad x_range")
    bx, by = x_dim // tx, y_dim // ty
    basis = dct_basis(n)
    m = measured_count(n)
    rows = x1 - x0
    P = rows * y_dim
    coeffs = np.empty((P, n))
    spectra = np.empty((P, n))
    masks = np.empty((P, m), dtype=np.uint8)
    y = np.empty((P, m))
    jobs = []
    for i in range(tx):
        lo, hi = max(x0, i * bx), min(x1, (i + 1) * bx)
        if lo >= hi:
            continue
        for j in range(ty):
            jobs.append((i, j, lo, hi))
    specs = [(bx * by, n, seed + ty * i + j) for i, j, _, _ in jobs]
    if workers > 1 and len(jobs) > 1:
        from concurrent.futures import ProcessPoolExecutor
        with ProcessPoolExecutor(max_workers=min(workers, len(jobs))) as pool:
            parts = list(pool.map(_tile_job, specs))
    else:
        parts = [_tile(n_pix, n, basis, s) for n_pix, _, s in specs]
    # pixel (ix, iy) -> flat index (ix - x0) * y_dim + iy (x-major, `solvers.py:497`)
    flat = np.arange(P).reshape(rows, y_dim)
    for (i, j, lo, hi), (c, f, mk, yy) in zip(jobs, parts):
        keep = slice((lo - i * bx) * by, (hi - i * bx) * by)   # tile rows lo..hi-1, all columns
        idx = flat[lo - x0:hi - x0, j * by:(j + 1) * by].reshape(-1)
        coeffs[idx], spectra[idx], masks[idx], y[idx] = c[keep], f[keep], mk[keep], yy[keep]
    return SyntheticCube(basis=basis, coeffs=coeffs, spectra=spectra, masks=masks, y=y,
                         shape=(rows, y_dim), seeds=tuple(s for _, _, s in specs))


@dataclass
class DeviceCube:
    """A synthetic cube generated on the GPU (generate_device): the same
    arrays as SyntheticCube, as CUDA tensors (coeffs only when requested)."""

    basis: np.ndarray
    spectra: object
    masks: object
    y: object
    coeffs: object
    shape: tuple
    seeds: tuple
    zero_fraction: float
    version: str = GENERATOR_VERSION

    @property
    def n(self):
        return int(self.basis.shape[0])

    @property
    def m(self):
        return int(self.masks.shape[1])

    @property
    def n_pixels(self):
        return int(self.y.shape[0])


def generate_device(x_dim, y_dim, n, seed=0, tiles=(1, 1), x_range=None, with_coeffs=False, workers=16,
                    device="cuda"):
    """`generate` with the input-side step on the GPU.

    The host only draws each tile's random stream (`_draw`, numpy, one thread
    per tile); the spectra (hcs_synth_spectra), the DCT, the T max|c|
    threshold, the reference spectra, the per-pixel masks (the M smallest
    keys) and the measurements (hcs_sparsify_measure) are computed on the
    device.  Same cube as `generate` up to FP64 rounding (exp and the DCT
    GEMMs sum in a different order; tests/test_gpu_input.py bounds it), with
    identical masks.
    """
    import torch
    from concurrent.futures import ThreadPoolExecutor

    from . import sparsify as sp

    if n > 256:
        raise ValueError("band indices are stored as uint8: n must be <= 256")
    tx, ty = tiles
    if x_dim % tx or y_dim % ty:
        raise ValueError("tiles must divide the cube")
    x0, x1 = x_range if x_range is not None else (0, x_dim)
    if not 0 <= x0 <= x1 <= x_dim:
        raise ValueError("bad x_range")
    bx, by = x_dim // tx, y_dim // ty
    basis = dct_basis(n)
    m = measured_count(n)
    rows = x1 - x0
    P = rows * y_dim
    dev = torch.device(device)
    basis_d = torch.as_tensor(basis, device=dev)
    spectra = torch.empty((P, n), dtype=torch.float64, device=dev)
    masks = torch.empty((P, m), dtype=torch.uint8, device=dev)
    y = torch.empty((P, m), dtype=torch.float64, device=dev)
    coeffs = torch.empty((P, n), dtype=torch.float64, device=dev) if with_coeffs else None
    jobs = [(i, j, max(x0, i * bx), min(x1, (i + 1) * bx)) for i in range(tx) for j in range(ty)]
    jobs = [jb for jb in jobs if jb[2] < jb[3]]
    seeds = [seed + ty * i + j for i, j, _, _ in jobs]
    flat = torch.arange(P, device=dev).reshape(rows, y_dim)
    zeroed = 0
    with ThreadPoolExecutor(max_workers=max(1, min(workers, len(jobs)))) as pool:
        draws = [pool.submit(_draw, bx * by, n, s) for s in seeds]
        for (i, j, lo, hi), fut in zip(jobs, draws):
            keep = slice((lo - i * bx) * by, (hi - i * bx) * by)   # tile rows lo..hi-1
            cen, wid, amp, noise, keys = (np.ascontiguousarray(a[keep]) for a in fut.result())
            f = sp.synth_spectra(*(torch.as_tensor(a, device=dev) for a in (cen, wid, amp, noise)))
            out = sp.sparsify_measure(f, basis_d, m, rule="maxrel", factor=SPARSIFY_T,
                                      keys=torch.as_tensor(keys, device=dev), with_coeffs=with_coeffs)
            idx = flat[lo - x0:hi - x0, j * by:(j + 1) * by].reshape(-1)
            spectra[idx], masks[idx], y[idx] = out.spectra, out.masks, out.y
            if with_coeffs:
                coeffs[idx] = out.coeffs
            zeroed += out.zeroed
            del f, out
    return DeviceCube(basis=basis, spectra=spectra, masks=masks, y=y, coeffs=coeffs, shape=(rows, y_dim),
                      seeds=tuple(seeds), zero_fraction=zeroed / float(max(P * n, 1)))


def generate_named_device(name, seed=0, x_range=None, with_coeffs=False, device="cuda"):
    spec = dict(CUBES[name])
    return generate_device(seed=seed, x_range=x_range, with_coeffs=with_coeffs, device=device, **spec)


# BASELINE.json configs (shape, bands, tiling)
CUBES = {
    "jasper": dict(x_dim=100, y_dim=100, n=198),                 # cfg1, cfg2
    "china": dict(x_dim=420, y_dim=140, n=154),                  # cfg3
    "salinas": dict(x_dim=512, y_dim=217, n=224),                # cfg4
    "scaling": dict(x_dim=2048, y_dim=868, n=224, tiles=(4, 4)),  # cfg5
}


def generate_named(name, seed=0, x_range=None, workers=1):
    spec = dict(CUBES[name])
    return generate(seed=seed, x_range=x_range, workers=workers, **spec)


def _strided_job(args):
    """Pixels of one tile whose global flat index is a multiple of `stride`."""
    n_pix, n, seed, i, j, bx, by, y_dim, stride = args
    c, f, mk, yy = _tile(n_pix, n, dct_basis(n), seed)
    t = np.arange(n_pix)
    p = (i * bx + t // by) * y_dim + j * by + t % by          # global x-major index
    keep = np.flatnonzero(p % stride == 0)
    return p[keep], c[keep], f[keep], mk[keep], yy[keep]


def generate_strided(name, stride=97, seed=0, workers=1):
    """Every `stride`-th pixel (global x-major index p with p % stride == 0) of
    a named cube, bit-identical to the same pixels of `generate_named` --
    the fixed deterministic subset the CPU baseline is timed on (SURVEY.md
    §8(d): "every 97th pixel").  Tiles are generated whole (the random stream
    is per tile) in a process pool and reduced to their sampled pixels.
    Returns a SyntheticCube of shape (S, 1) in increasing p order; its
    ``seeds`` holds the tile seeds and ``pixel_index`` the global indices."""
    spec = dict(CUBES[name])
    x_dim, y_dim, n = spec["x_dim"], spec["y_dim"], spec["n"]
    tx, ty = spec.get("tiles", (1, 1))
    bx, by = x_dim // tx, y_dim // ty
    jobs = [(bx * by, n, seed + ty * i + j, i, j, bx, by, y_dim, stride) for i in range(tx) for j in range(ty)]
    if workers > 1 and len(jobs) > 1:
        from concurrent.futures import ProcessPoolExecutor
        with ProcessPoolExecutor(max_workers=min(workers, len(jobs))) as pool:
            parts = list(pool.map(_strided_job, jobs))
    else:
        parts = [_strided_job(jb) for jb in jobs]
    p = np.concatenate([pt[0] for pt in parts])
    order = np.argsort(p, kind="stable")
    cat = [np.concatenate([pt[k] for pt in parts])[order] for k in range(1, 5)]
    cube = SyntheticCube(basis=dct_basis(n), coeffs=cat[0], spectra=cat[1], masks=cat[2],
                         y=np.ascontiguousarray(cat[3]), shape=(len(p), 1),
                         seeds=tuple(jb[2] for jb in jobs))
    cube.pixel_index = p[order]
    return cube
