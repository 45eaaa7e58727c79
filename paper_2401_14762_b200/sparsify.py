"""Input side of the recovery pipeline on the GPU.

The reference prepares a cube in two CLI stages: `run_sparsify`
(`cli.py:97-126`) maps every pixel spectrum to the sparse domain
(`to_sparse_domain`, `transform.py:40-45`), zeroes small coefficients
(`sparsify`, `transform.py:73-97`: keep (|x| - mean|x|) >= factor * std|x|)
and maps back (`from_sparse_domain`, `transform.py:48-60`); `run_compress`
(`cli.py:129-139`) then keeps a seeded subset of bands (`measure`,
`transform.py:168-173`).  Here both stages are one kernel over 32-pixel
tiles for the orthonormal DCT-II and per-pixel masks (BASELINE.json's
model), with the reference's mean/std rule ("meanstd") or the BASELINE
generator's |c| < T max|c| rule ("maxrel").

Inputs may be numpy arrays (copied to the device) or CUDA tensors; results
are CUDA tensors.  Everything runs in libhypercs_b200.so (no host fallback).
"""

from dataclasses import dataclass

import numpy as np

from . import _native as nat

RULES = {"maxrel": 0, "meanstd": 1}


def _torch():
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("libhypercs_b200 needs a CUDA device (no CPU fallback)")
    return torch


def _dev(a, dtype):
    torch = _torch()
    if isinstance(a, torch.Tensor):
        return a.to(device="cuda", dtype=dtype).contiguous()
    return torch.as_tensor(np.ascontiguousarray(a), device="cuda").to(dtype)


@dataclass
class Measured:
    """Result of sparsify_measure (pixel-major CUDA tensors).

    spectra  (P, N) sparsified spectra f_s = Psi c_s (the PSNR reference)
    coeffs   (P, N) kept DCT coefficients c_s, or None
    masks    (P, M) uint8 sorted measured band indices
    y        (P, M) measurements f_s[mask]
    zeroed   number of coefficients set to zero (zero_fraction = zeroed / (P N))
    """

    spectra: object
    coeffs: object
    masks: object
    y: object
    zeroed: int

    @property
    def zero_fraction(self):
        P, N = self.spectra.shape
        return self.zeroed / float(max(P * N, 1))


def synth_spectra(centres, widths, amps, noise):
    """Spectra of the frozen synthetic generator (synth.py v1) from its drawn
    parameters: clip(sum_i amps_i exp(-((b - centres_i) / widths_i)^2 / 2)
    + noise, 0, 1); centres/widths/amps (P, 4), noise (P, N)."""
    torch = _torch()
    c, w, a, z = (_dev(v, torch.float64) for v in (centres, widths, amps, noise))
    P, N = z.shape
    if c.shape != (P, 4) or w.shape != (P, 4) or a.shape != (P, 4):
        raise ValueError("centres/widths/amps must be (P, 4)")
    f = torch.empty_like(z)
    nat.check(nat.load().hcs_synth_spectra(P, N, nat.ptr(c), nat.ptr(w), nat.ptr(a), nat.ptr(z), nat.ptr(f),
                                           nat.stream_handle()))
    return f


def sparsify_measure(spectra, basis, m, rule="meanstd", factor=1.0, masks=None, keys=None, with_coeffs=True,
                     with_spectra=True):
    """Sparsify every pixel spectrum in the DCT domain and measure it.

    spectra (P, N); basis the orthonormal synthesis matrix Psi (N, N);
    m measured bands per pixel.  Masks come from `masks` (P, m) or, with
    `keys` (P, N), are the m smallest keys' band indices (sorted).
    factor < 0 raises ValueError (transform.py:85-86).
    """
    torch = _torch()
    if rule not in RULES:
        raise ValueError(f"unknown threshold rule {rule!r}")
    if factor < 0:
        raise ValueError("threshold factor must be >= 0")
    f = _dev(spectra, torch.float64)
    if f.dim() != 2:
        raise ValueError("spectra must be (P, N)")
    P, N = f.shape
    b = _dev(basis, torch.float64)
    if b.shape != (N, N):
        raise ValueError("basis must be N x N")
    if not 1 <= m <= N:
        raise ValueError("m must be in [1, N]")
    if (masks is None) == (keys is None):
        raise ValueError("give exactly one of masks, keys")
    if keys is not None:
        k = _dev(keys, torch.float64)
        if k.shape != (P, N):
            raise ValueError("keys must be (P, N)")
        mk = torch.empty((P, m), dtype=torch.uint8, device="cuda")
    else:
        k = None
        mk = _dev(masks, torch.uint8)
        if mk.shape != (P, m):
            raise ValueError("masks must be (P, m)")
    y = torch.empty((P, m), dtype=torch.float64, device="cuda")
    cf = torch.empty((P, N), dtype=torch.float64, device="cuda") if with_coeffs else None
    fs = torch.empty((P, N), dtype=torch.float64, device="cuda") if with_spectra else None
    nz = torch.zeros(1, dtype=torch.int64, device="cuda")
    nat.check(nat.load().hcs_sparsify_measure(P, N, m, nat.ptr(b), nat.ptr(f), RULES[rule], float(factor),
                                              nat.ptr(k), nat.ptr(mk), nat.ptr(cf), nat.ptr(fs), nat.ptr(y),
                                              nat.ptr(nz), nat.stream_handle()))
    return Measured(spectra=fs, coeffs=cf, masks=mk, y=y, zeroed=int(nz.item()))
