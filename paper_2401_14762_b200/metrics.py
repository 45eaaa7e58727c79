"""Quality metrics on the recovery output (`hypercs/metrics.py:30-64`).

`psnr` keeps the reference's semantics (abs-max peak over the reference cube,
mean squared error over all voxels, inf when identical); `psnr_from_coeffs`
is the device path used by the benchmark: it reconstructs spectra Psi x on
the fly inside the PSNR kernel (no spectra cube is materialised) and returns
the partial sums so ranks can all-reduce them (one NCCL all-reduce).
"""

import math

import numpy as np

from . import _native as nat

PEAK_CONVENTIONS = ("abs-max", "signed-max", "range")


class UndefinedMetricError(ValueError):
    """The metric is undefined for these inputs (e.g. an all-zero reference)."""


def psnr(reference, reconstruction, peak="abs-max"):
    """PSNR in dB between two cubes (metrics.py:30-55); arrays or objects with .data."""
    ref = np.asarray(getattr(reference, "data", reference))
    rec = np.asarray(getattr(reconstruction, "data", reconstruction))
    if ref.shape != rec.shape:
        raise ValueError(f"cube shapes differ: {ref.shape} vs {rec.shape}")
    if peak == "abs-max":
        peak_value = float(np.abs(ref).max())
    elif peak == "signed-max":
        peak_value = float(ref.max())
    elif peak == "range":
        peak_value = float(ref.max() - ref.min())
    else:
        raise ValueError(f"unknown peak convention {peak!r}")
    if peak_value <= 0:
        raise UndefinedMetricError(f"non-positive peak {peak_value} under {peak!r}")
    mse = float(np.mean((ref - rec) ** 2))
    if mse == 0.0:
        return math.inf
    return 10.0 * math.log10(peak_value * peak_value / mse)


def psnr_partials(ref_spectra, coeffs, basis, out=None, stream=None):
    """Device partial sums [SSE, max|ref|] of ref vs Psi @ x over P x n (CUDA tensors).

    Accumulates into ``out`` (a float64[2] CUDA tensor) when given."""
    import torch
    P, n = int(ref_spectra.shape[0]), int(ref_spectra.shape[1])
    if out is None:
        out = torch.zeros(2, dtype=torch.float64, device=ref_spectra.device)
    nat.check(nat.load().hcs_psnr_partials(P, n, nat.ptr(ref_spectra), nat.ptr(coeffs), nat.ptr(basis),
                                           ctypes_ptr(out, 0), ctypes_ptr(out, 1), nat.stream_handle(stream)))
    return out


def sse_coeff_partials(ref_coeffs, coeffs, out=None, stream=None):
    """Device SSE of the recovered spectra in the coefficient domain (CUDA tensors).

    For the orthonormal DCT-II basis ||f_ref - Psi x||^2 = ||c_ref - x||^2
    (Parseval), so PSNR needs only the sparsified reference coefficients and the
    recovered ones: one HBM stream (hcs_sse_coeff_partials), no spectra GEMM.
    Accumulates into ``out[0]`` (a float64 CUDA tensor) when given."""
    import torch
    if ref_coeffs.shape != coeffs.shape or ref_coeffs.dtype != torch.float64 or coeffs.dtype != torch.float64:
        raise ValueError("ref_coeffs and coeffs must be float64 arrays of the same shape")
    if not (ref_coeffs.is_contiguous() and coeffs.is_contiguous()):
        raise ValueError("ref_coeffs and coeffs must be contiguous")
    P, n = int(ref_coeffs.shape[0]), int(ref_coeffs.shape[1])
    if out is None:
        out = torch.zeros(1, dtype=torch.float64, device=ref_coeffs.device)
    nat.check(nat.load().hcs_sse_coeff_partials(P, n, nat.ptr(ref_coeffs), nat.ptr(coeffs), ctypes_ptr(out, 0),
                                                nat.stream_handle(stream)))
    return out


def ctypes_ptr(t, i):
    import ctypes
    return ctypes.c_void_p(t.data_ptr() + i * t.element_size())


def psnr_from_partials(sse, peak, count):
    if peak <= 0:
        raise UndefinedMetricError(f"non-positive peak {peak} under 'abs-max'")
    mse = sse / count
    return math.inf if mse == 0.0 else 10.0 * math.log10(peak * peak / mse)


def psnr_from_coeffs(ref_spectra, coeffs, basis):
    """PSNR of the spectra Psi x against the reference spectra (device tensors)."""
    part = psnr_partials(ref_spectra, coeffs, basis).cpu().numpy()
    return psnr_from_partials(float(part[0]), float(part[1]), ref_spectra.numel())


def convergence_ratio(results):
    """Percentage of converged pixels; None entries count as not converged (metrics.py:58-64)."""
    results = list(results)
    if not results:
        raise ValueError("no solver results to aggregate")
    converged = sum(1 for r in results if r is not None and r.converged)
    return 100.0 * converged / len(results)
