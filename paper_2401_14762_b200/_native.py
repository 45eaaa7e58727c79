"""ctypes binding of libhypercs_b200.so (the C ABI in include/hypercs_b200.h).

The shared library is built in-tree by `__graft_entry__.build()` (nvcc,
sm_100a).  There is no fallback: if the library is missing or no CUDA device
is present, every call raises.  Device memory and streams come from PyTorch
(plumbing only); the compute is the library's hand-written kernels.
"""

import ctypes
import os
from pathlib import Path

LIB_NAME = "libhypercs_b200.so"
LIB_PATH = Path(__file__).resolve().parent / LIB_NAME

HCS_OK, HCS_EINVAL, HCS_ECUDA, HCS_ENONFINITE = 0, 1, 2, 3
ALGO_IDS = {"fista": 0, "admm": 1, "gomp": 2, "biht": 3, "cosamp": 4}

EXPORTS = (
    "hcs_abi_version", "hcs_last_error", "hcs_workspace_bytes", "hcs_recover", "hcs_recover_status",
    "hcs_soft_threshold", "hcs_argmax_k", "hcs_least_squares", "hcs_residual_delta", "hcs_lipschitz",
    "hcs_psnr_partials", "hcs_dmma_peak_tflops", "hcs_synth_spectra", "hcs_sparsify_measure",
    "hcs_sse_coeff_partials", "hcs_recover_launches", "hcs_check_basis", "hcs_checked_build",
)


class HcsParams(ctypes.Structure):
    _fields_ = [
        ("lam", ctypes.c_double),
        ("mu", ctypes.c_double),
        ("alpha", ctypes.c_double),
        ("epsilon", ctypes.c_double),
        ("kappa", ctypes.c_int32),
        ("atoms_per_iter", ctypes.c_int32),
        ("max_iter", ctypes.c_int32),
        ("reserved", ctypes.c_int32),
        ("time_limit", ctypes.c_double),
    ]


class HcsStats(ctypes.Structure):
    _fields_ = [
        ("iterations", ctypes.c_void_p),
        ("converged", ctypes.c_void_p),
        ("final_delta", ctypes.c_void_p),
        ("failed_at", ctypes.c_void_p),
        ("admm_gap", ctypes.c_void_p),
        ("lipschitz", ctypes.c_void_p),
        ("elapsed", ctypes.c_void_p),
        ("work", ctypes.c_void_p),
        ("trace", ctypes.c_void_p),
        ("trace_len", ctypes.c_void_p),
        ("trace_calls", ctypes.c_int32),
        ("reserved", ctypes.c_int32),
    ]


_lib = None


def load(path=None):
    """Load the library (once).  Raises RuntimeError if it was not built."""
    global _lib
    if _lib is not None:
        return _lib
    p = Path(path or os.environ.get("HCS_LIB", LIB_PATH))
    if not p.exists():
        raise RuntimeError(
            f"{p} is missing: the CUDA library is required (no CPU fallback); "
            "build it with `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = ctypes.CDLL(str(p))
    vp, i64, i32, dbl = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_double
    lib.hcs_abi_version.restype = ctypes.c_int
    lib.hcs_last_error.restype = ctypes.c_char_p
    lib.hcs_workspace_bytes.restype = ctypes.c_size_t
    lib.hcs_workspace_bytes.argtypes = [ctypes.c_int, i64, i32, i32]
    lib.hcs_recover.restype = ctypes.c_int
    lib.hcs_recover.argtypes = [ctypes.c_int, i64, i32, i32, vp, vp, vp, ctypes.POINTER(HcsParams), vp,
                                ctypes.POINTER(HcsStats), vp, ctypes.c_size_t, vp]
    lib.hcs_check_basis.restype = ctypes.c_int
    lib.hcs_check_basis.argtypes = [i32, vp, ctypes.POINTER(ctypes.c_double), vp]
    lib.hcs_recover_launches.restype = ctypes.c_int
    lib.hcs_recover_launches.argtypes = [ctypes.c_int, i32, i32, ctypes.POINTER(HcsParams)]
    lib.hcs_recover_status.restype = ctypes.c_int
    lib.hcs_recover_status.argtypes = [vp, vp]
    lib.hcs_soft_threshold.argtypes = [i64, vp, dbl, vp, vp]
    lib.hcs_argmax_k.argtypes = [i64, i32, vp, i32, vp, vp]
    lib.hcs_least_squares.argtypes = [i64, i32, i32, vp, vp, vp, vp, vp]
    lib.hcs_residual_delta.argtypes = [i64, i32, vp, vp, vp, vp]
    lib.hcs_lipschitz.argtypes = [i64, i32, i32, vp, vp, vp, vp]
    lib.hcs_psnr_partials.argtypes = [i64, i32, vp, vp, vp, vp, vp, vp]
    lib.hcs_sse_coeff_partials.argtypes = [i64, i32, vp, vp, vp, vp]
    lib.hcs_synth_spectra.argtypes = [i64, i32, vp, vp, vp, vp, vp, vp]
    lib.hcs_sparsify_measure.argtypes = [i64, i32, i32, vp, vp, i32, dbl, vp, vp, vp, vp, vp, vp, vp]
    lib.hcs_dmma_peak_tflops.argtypes = [ctypes.POINTER(ctypes.c_double), ctypes.c_int]
    lib.hcs_dmma_peak_tflops.restype = ctypes.c_int
    for name in ("hcs_soft_threshold", "hcs_argmax_k", "hcs_least_squares", "hcs_residual_delta",
                 "hcs_lipschitz", "hcs_psnr_partials", "hcs_synth_spectra", "hcs_sparsify_measure",
                 "hcs_sse_coeff_partials"):
        getattr(lib, name).restype = ctypes.c_int
    _lib = lib
    return lib


def check(code):
    """Map an ABI return code to the reference's exception types."""
    if code == HCS_OK:
        return
    msg = load().hcs_last_error().decode()
    if code in (HCS_EINVAL, HCS_ENONFINITE):
        raise ValueError(msg)
    raise RuntimeError(f"CUDA error in libhypercs_b200: {msg}")


def ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else ctypes.c_void_p(0)


def stream_handle(stream=None):
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def dmma_peak_tflops(iters=20000):
    """Measured FP64 DMMA peak of the current GPU (TFLOP/s)."""
    out = ctypes.c_double(0.0)
    if load().hcs_dmma_peak_tflops(ctypes.byref(out), iters) != 0:
        raise RuntimeError("dmma peak microbenchmark failed")
    return out.value
