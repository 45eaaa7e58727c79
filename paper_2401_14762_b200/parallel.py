"""Multi-GPU sharding of a cube recovery (one process per GPU).

Pixels are independent (the reference's only parallelism is a process pool
over pixels, `solvers.py:487-493`), so a cube is split into contiguous slabs
of x-rows (the leading axis of the x-major (X, Y, .) arrays, `cube.py:62`,
`solvers.py:497`), one per rank, with no data-path communication.  The only
collective is one all-reduce of the per-configuration sums that make the
cube-level statistics (PSNR SSE, n_converged, n_failed, n_zero,
total_iterations; `metrics.py:30-64`, `solvers.py:503-513`); the PSNR peak is
input-derived and reduced once at setup (MAX).

Works with any torch.distributed backend: NCCL over NVLink on the B200s,
gloo on CPU for the tests.
"""

import math

STAT_FIELDS = ("sse", "n_converged", "n_failed", "n_zero_pixels", "total_iterations", "work_flops")


def row_slab(x_dim, rank, world):
    """[x0, x1) rows of rank `rank` out of `world` (balanced, contiguous)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    return rank * x_dim // world, (rank + 1) * x_dim // world


def local_stats(batch, ok_mask=None):
    """[n_converged, n_failed, n_zero_pixels, total_iterations, work] of one
    DeviceBatch (or any object with iterations/converged/failed_at tensors and
    optionally work), as in RecoveryStats (solvers.py:503-513)."""
    ok = batch.failed_at < 0
    conv = batch.converged.bool()
    work = getattr(batch, "work", None)
    return [
        (conv & ok).sum(),
        (~ok).sum(),
        ((batch.iterations == 0) & conv & ok).sum(),
        batch.iterations[ok].sum(),
        work.sum() if work is not None else 0.0,
    ]


def all_reduce_stats(stats, group=None):
    """Sum a (configs, len(STAT_FIELDS)) float64 tensor over all ranks in place."""
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(stats, op=dist.ReduceOp.SUM, group=group)
    return stats


def all_reduce_max(t, group=None):
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return t


def cube_summary(row, peak, n_pixels, n_bands):
    """Cube-level numbers from one reduced STAT_FIELDS row (metrics.py:30-64)."""
    sse, conv, failed, zero, iters = (float(v) for v in row[:5])
    mse = sse / (n_pixels * n_bands)
    return {
        "psnr_db": math.inf if mse == 0 else 10.0 * math.log10(peak * peak / mse),
        "convergence_pct": 100.0 * conv / n_pixels,
        "n_converged": int(conv),
        "n_failed": int(failed),
        "n_zero_pixels": int(zero),
        "total_iterations": int(iters),
    }
