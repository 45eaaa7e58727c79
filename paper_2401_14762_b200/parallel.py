"""Multi-GPU sharding of a cube recovery (one process per GPU).

Pixels are independent (the reference's only parallelism is a process pool
over pixels, `solvers.py:487-493`), so a cube is split into contiguous slabs
of x-rows (the leading axis of the x-major (X, Y, .) arrays, `cube.py:62`,
`solvers.py:497`), one per rank, with no data-path communication.  The only
collective is one all-reduce of the per-configuration sums that make the
cube-level statistics (PSNR SSE, n_converged, n_failed, n_zero,
total_iterations, work; `metrics.py:30-64`, `solvers.py:503-513`); the PSNR
peak is input-derived and reduced once at setup (MAX).

Pieces:
  * `spawn_ranks` -- re-launch a script as N ranks under torch.distributed.run
    (127.0.0.1 rendezvous, one process per GPU); `bench.py --gpus N` uses it;
  * `init_from_env` -- RANK / WORLD_SIZE / LOCAL_RANK and the process group;
  * `ShardedStep` -- one step over this rank's slab: every solver
    configuration, its PSNR partial and statistics, then the one all-reduce
    (the bench's timed step; the solve / SSE functions are injectable so the
    CPU tests drive the same step with a fake solve over gloo);
  * `recover_cube_sharded` -- the API form: `recover_cube` on this rank's slab
    of a host cube plus the reduced cube-level statistics.

Works with any torch.distributed backend: NCCL over NVLink on the B200s,
gloo on CPU for the tests.
"""

import math
import os
import socket
import subprocess
import sys

STAT_FIELDS = ("sse", "n_converged", "n_failed", "n_zero_pixels", "total_iterations", "work_flops")


def row_slab(x_dim, rank, world):
    """[x0, x1) rows of rank `rank` out of `world` (balanced, contiguous)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    return rank * x_dim // world, (rank + 1) * x_dim // world


def free_port():
    with socket.socket(socket.AF_INET, socket.SOCK_STREAM) as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def spawn_ranks(nprocs, argv, env=None, port=None):
    """Run ``python argv...`` as `nprocs` ranks of one node under
    torch.distributed.run (rendezvous on 127.0.0.1); returns the exit code.
    Each rank sees RANK / LOCAL_RANK / WORLD_SIZE / MASTER_ADDR / MASTER_PORT."""
    if nprocs < 1:
        raise ValueError("nprocs must be >= 1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nprocs}",
           "--master-addr=127.0.0.1", f"--master-port={port or free_port()}", *argv]
    full_env = dict(os.environ)
    full_env.update(env or {})
    return subprocess.call(cmd, env=full_env)


def dist_env():
    """(rank, world, local_rank) from the launcher's environment (1 process: 0, 1, 0)."""
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def init_from_env(backend="nccl", device=None):
    """Initialise the default process group when WORLD_SIZE > 1; returns (rank, world, local_rank)."""
    import torch.distributed as dist
    rank, world, local = dist_env()
    if world > 1 and not dist.is_initialized():
        kw = {"device_id": device} if (backend == "nccl" and device is not None) else {}
        dist.init_process_group(backend, **kw)
    return rank, world, local


def _world(group=None):
    import torch.distributed as dist
    return dist.get_world_size(group) if dist.is_available() and dist.is_initialized() else 1


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
    if _world(group) > 1:
        dist.all_reduce(stats, op=dist.ReduceOp.SUM, group=group)
    return stats


def all_reduce_max(t, group=None):
    import torch.distributed as dist
    if _world(group) > 1:
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


class ShardedStep:
    """One step of a sharded cube recovery on this rank's slab.

    ``cfgs``: [(algorithm, SolverConfig)]; ``y`` (P, m), ``masks`` (P, m),
    ``basis`` (n, n) and ``coeffs`` (P, n, the reference coefficients for the
    coefficient-domain PSNR) are this rank's arrays.  Calling the step solves
    the slab with every configuration (``solve(algo, y, masks, basis, cfg,
    out=...)``, default `solvers.solve_batch` asynchronous), adds each
    configuration's SSE (``sse(coeffs, x, out=...)``, default
    `metrics.sse_coeff_partials`) and statistics into ``stats`` (configs x
    STAT_FIELDS), copies each launch's non-finite flag into ``errors`` and
    all-reduces ``stats`` once.  Returns the number of our kernel launches.
    ``record``: optional per-config (start, end) CUDA events."""

    def __init__(self, cfgs, y, masks, basis, coeffs, solve=None, sse=None, group=None):
        import torch
        if solve is None:
            from .solvers import solve_batch

            def solve(algo, y_, m_, b_, cfg, out=None):
                return solve_batch(algo, y_, m_, b_, cfg, check_status=False, out=out)
        if sse is None:
            from .metrics import sse_coeff_partials as sse
        self.cfgs, self.y, self.masks, self.basis, self.coeffs = list(cfgs), y, masks, basis, coeffs
        self.solve, self.sse, self.group = solve, sse, group
        dev = y.device
        self.stats = torch.zeros((len(self.cfgs), len(STAT_FIELDS)), dtype=torch.float64, device=dev)
        self.psnr = torch.zeros((len(self.cfgs), 1), dtype=torch.float64, device=dev)
        self.errors = torch.zeros((len(self.cfgs),), dtype=torch.int32, device=dev)
        self.out = None
        self.launches = 0

    def __call__(self, record=None):
        launches = 0
        self.psnr.zero_()
        for i, (algo, cfg) in enumerate(self.cfgs):
            if record is not None:
                record[i][0].record()
            b = self.solve(algo, self.y, self.masks, self.basis, cfg, out=self.out)
            if record is not None:
                record[i][1].record()
            self.out = b
            flag = b.error_flag() if hasattr(b, "error_flag") else None
            if flag is not None:
                self.errors[i].copy_(flag[0])
            # PSNR's squared error in the coefficient domain (Parseval)
            self.sse(self.coeffs, b.x, out=self.psnr[i, :1])
            for f, v in enumerate(local_stats(b)):
                self.stats[i, 1 + f] = v
            launches += getattr(b, "launches", 0) + 1
        self.stats[:, 0] = self.psnr[:, 0]
        all_reduce_stats(self.stats, self.group)   # the one data-path collective
        self.launches = launches
        return launches

    def check_errors(self):
        """ValueError if any configuration saw non-finite measurements (syncs)."""
        flags = self.errors.tolist()
        if any(f & 2 for f in flags):
            raise ValueError("mask entries must be strictly increasing band indices < N")
        bad = [self.cfgs[i][0] for i, f in enumerate(flags) if f]
        if bad:
            raise ValueError(f"array must not contain infs or NaNs ({', '.join(bad)})")


def recover_cube_sharded(measurements, dictionary, config, algorithm, group=None, **kwargs):
    """`recover_cube` (solvers.py:455-514) on this rank's x-row slab of a host
    cube, with the cube-level statistics reduced over the process group.

    ``measurements``: the whole (X, Y, m) cube (every rank passes the same
    array; only its slab is copied to this rank's GPU); ``dictionary``: a
    `Dictionary` with a shared mask or per-pixel masks for the whole cube.
    Returns ((x0, x1), slab cube (x1 - x0, Y, n), summary) where summary holds
    the whole cube's n_pixels / n_converged / n_failed / n_zero_pixels /
    total_iterations / recovery_time_s (sums over ranks) and this rank's
    RecoveryStats under "local"."""
    import numpy as np
    import torch
    from .solvers import recover_cube
    from .transform import Dictionary
    rank = 0
    world = _world(group)
    if world > 1:
        import torch.distributed as dist
        rank = dist.get_rank(group)
    x_dim, y_dim = int(measurements.shape[0]), int(measurements.shape[1])
    x0, x1 = row_slab(x_dim, rank, world)
    slab = measurements[x0:x1]
    if not isinstance(dictionary, Dictionary):
        dictionary = Dictionary.from_matrix(dictionary.matrix)
    if dictionary.shared:
        dic = dictionary
    else:
        masks = np.asarray(dictionary.masks).reshape(x_dim, y_dim, -1)[x0:x1].reshape(-1, dictionary.m)
        dic = Dictionary.per_pixel(dictionary.basis, masks)
    cube, st = recover_cube(slab, dic, config, algorithm, **kwargs)
    dev = torch.device("cuda", torch.cuda.current_device()) if torch.cuda.is_available() else torch.device("cpu")
    tot = torch.tensor([st.n_pixels, st.n_converged, st.n_failed, st.n_zero_pixels, st.total_iterations,
                        st.recovery_time_s], dtype=torch.float64, device=dev)
    if world > 1:
        import torch.distributed as dist
        dist.all_reduce(tot, op=dist.ReduceOp.SUM, group=group)
    t = tot.cpu().tolist()
    summary = {"n_pixels": int(t[0]), "n_converged": int(t[1]), "n_failed": int(t[2]), "n_zero_pixels": int(t[3]),
               "total_iterations": int(t[4]), "recovery_time_s": t[5], "local": st}
    return (x0, x1), cube, summary
