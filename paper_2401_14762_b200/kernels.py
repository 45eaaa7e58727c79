"""GPU forms of the reference's numeric kernels (`hypercs/kernels.py:14-85`).

Same names and argument meaning as the reference; inputs may be numpy arrays
(copied to the device, result copied back) or CUDA tensors (result stays on
the device).  Batched variants take a leading pixel axis.  Everything runs in
libhypercs_b200.so; there is no host fallback.
"""

import numpy as np

from . import _native as nat

RANK_RTOL = 1e-10   # kernels.py:11


def _torch():
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("libhypercs_b200 needs a CUDA device (no CPU fallback)")
    return torch


def _to_dev(a, dtype):
    torch = _torch()
    if isinstance(a, torch.Tensor):
        return a.to(device="cuda", dtype=dtype).contiguous(), True
    arr = np.asarray(a)
    if np.iscomplexobj(arr):
        if np.any(arr.imag != 0):
            raise ValueError("the GPU backend is real-valued")
        arr = arr.real
    return torch.as_tensor(np.ascontiguousarray(arr), device="cuda").to(dtype), False


def _out(t, on_device):
    return t if on_device else t.cpu().numpy()


def soft_threshold(v, t):
    """v * max(|v| - t, 0) / |v|, exact 0 where |v| <= t (kernels.py:14-28)."""
    if t < 0:
        raise ValueError("threshold must be >= 0")
    torch = _torch()
    dv, dev = _to_dev(v, torch.float64)
    out = torch.empty_like(dv)
    nat.check(nat.load().hcs_soft_threshold(dv.numel(), nat.ptr(dv), float(t), nat.ptr(out), nat.stream_handle()))
    return _out(out, dev)


def argmax_k(v, k):
    """Indexes of the k largest |v| (ties to the lowest index), ascending
    (kernels.py:31-41).  A 2-D input is treated as a batch of rows."""
    torch = _torch()
    dv, dev = _to_dev(v, torch.float64)
    rows = dv.reshape(1, -1) if dv.dim() == 1 else dv
    n = rows.shape[1]
    if not 1 <= k <= n:
        raise ValueError(f"k must be in [1, {n}], got {k}")
    if n > 256:
        raise ValueError("argmax_k on the GPU supports length <= 256")
    idx = torch.empty((rows.shape[0], k), dtype=torch.int32, device="cuda")
    nat.check(nat.load().hcs_argmax_k(rows.shape[0], n, nat.ptr(rows), k, nat.ptr(idx), nat.stream_handle()))
    idx = idx.to(torch.int64)
    if dv.dim() == 1:
        idx = idx[0]
    return _out(idx, dev)


def least_squares(b, y, return_path=False):
    """min_s ||b s - y|| by column-pivoted QR with the minimum-norm fallback
    below RANK_RTOL (kernels.py:44-67).  b: (m, k) or (P, m, k)."""
    torch = _torch()
    db, dev = _to_dev(b, torch.float64)
    dy, _ = _to_dev(y, torch.float64)
    if db.dim() not in (2, 3):
        raise ValueError("matrix must be 2-D")
    single = db.dim() == 2
    if single:
        db, dy = db.unsqueeze(0), dy.reshape(1, -1)
    P, m, k = db.shape
    if dy.shape != (P, m):
        raise ValueError("right-hand side length does not match the matrix")
    s = torch.empty((P, k), dtype=torch.float64, device="cuda")
    path = torch.empty((P,), dtype=torch.int32, device="cuda")
    nat.check(nat.load().hcs_least_squares(P, m, k, nat.ptr(db.contiguous()), nat.ptr(dy.contiguous()),
                                           nat.ptr(s), nat.ptr(path), nat.stream_handle()))
    if single:
        s, path = s[0], path[0]
    s = _out(s, dev)
    return (s, _out(path, dev)) if return_path else s


def residual_delta(r, r_prev):
    """||r - r_prev||_2 (kernels.py:70-76); batched over a leading axis."""
    torch = _torch()
    dr, dev = _to_dev(r, torch.float64)
    dp, _ = _to_dev(r_prev, torch.float64)
    if dr.shape != dp.shape:
        raise ValueError("residual lengths differ")
    rows = dr.reshape(1, -1) if dr.dim() == 1 else dr
    prow = dp.reshape(1, -1) if dp.dim() == 1 else dp
    out = torch.empty((rows.shape[0],), dtype=torch.float64, device="cuda")
    nat.check(nat.load().hcs_residual_delta(rows.shape[0], rows.shape[1], nat.ptr(rows.contiguous()),
                                            nat.ptr(prow.contiguous()), nat.ptr(out), nat.stream_handle()))
    if dr.dim() == 1:
        return float(out[0].item())
    return _out(out, dev)


def gather_columns(a, support):
    """Columns of a (or a.matrix) at the support indexes (kernels.py:79-85)."""
    matrix = a.matrix if hasattr(a, "matrix") else np.asarray(a)
    support = np.asarray(support, dtype=np.intp)
    if support.size and (support.min() < 0 or support.max() >= matrix.shape[1]):
        raise IndexError("support index out of range")
    return matrix[:, support]


def lipschitz_batch(basis, masks):
    """Power-iteration Lipschitz constants of A_p = basis[masks[p], :] (GPU)."""
    torch = _torch()
    db, _ = _to_dev(basis, torch.float64)
    dm = torch.as_tensor(np.ascontiguousarray(masks, dtype=np.uint8), device="cuda")
    P, m = dm.shape
    out = torch.empty((P,), dtype=torch.float64, device="cuda")
    nat.check(nat.load().hcs_lipschitz(P, db.shape[0], m, nat.ptr(db), nat.ptr(dm), nat.ptr(out),
                                       nat.stream_handle()))
    return out.cpu().numpy()
