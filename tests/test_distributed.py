"""Multi-process sharding on CPU (gloo, world size 2): row slabs cover the cube
exactly once and the one all-reduce of per-configuration sums reproduces the
single-process statistics (paper_2401_14762_b200.parallel)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2401_14762_b200 import parallel


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


class _Batch:
    def __init__(self, it, conv, failed):
        self.iterations = torch.as_tensor(it, dtype=torch.int32)
        self.converged = torch.as_tensor(conv, dtype=torch.uint8)
        self.failed_at = torch.as_tensor(failed, dtype=torch.int32)


def _fake_results(P, seed=0):
    rng = np.random.default_rng(seed)
    it = rng.integers(0, 50, size=P).astype(np.int32)
    conv = (rng.random(P) < 0.9).astype(np.uint8)
    failed = np.where(rng.random(P) < 0.05, 1, -1).astype(np.int32)
    sq = rng.random(P)
    return it, conv, failed, sq


def _worker(rank, world, port, X, Y, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    it, conv, failed, sq = _fake_results(X * Y)
    x0, x1 = parallel.row_slab(X, rank, world)
    sl = slice(x0 * Y, x1 * Y)
    b = _Batch(it[sl], conv[sl], failed[sl])
    stats = torch.zeros((1, len(parallel.STAT_FIELDS)), dtype=torch.float64)
    stats[0, 0] = float(sq[sl].sum())
    for f, v in enumerate(parallel.local_stats(b)):
        stats[0, 1 + f] = v
    parallel.all_reduce_stats(stats)
    peak = parallel.all_reduce_max(torch.tensor([float(sq[sl].max())], dtype=torch.float64))
    if rank == 0:
        out.put((stats.numpy().tolist(), float(peak[0]), (x0, x1)))
    dist.barrier()
    dist.destroy_process_group()


def test_row_slabs_partition_the_cube():
    for X in (1, 7, 100, 2048):
        for world in (1, 2, 3, 8):
            if world > X:
                continue
            slabs = [parallel.row_slab(X, r, world) for r in range(world)]
            assert slabs[0][0] == 0 and slabs[-1][1] == X
            assert all(a[1] == b[0] for a, b in zip(slabs, slabs[1:]))
            sizes = [b - a for a, b in slabs]
            assert max(sizes) - min(sizes) <= 1


def test_gloo_world2_reduction_matches_single_process():
    X, Y = 9, 7
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, X, Y, q)) for r in range(2)]
    for p in procs:
        p.start()
    stats, peak, _ = q.get(timeout=90)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    it, conv, failed, sq = _fake_results(X * Y)
    ok = failed < 0
    expect = [sq.sum(), (conv.astype(bool) & ok).sum(), (~ok).sum(),
              ((it == 0) & conv.astype(bool) & ok).sum(), it[ok].sum(), 0.0]
    np.testing.assert_allclose(stats[0], expect, rtol=1e-12)
    assert peak == pytest.approx(sq.max())
    summ = parallel.cube_summary(stats[0], 1.0, X * Y, 4)
    assert summ["n_failed"] == int((~ok).sum())


def test_launcher_drives_sharded_step_world2(tmp_path):
    """bench.py's launcher (parallel.spawn_ranks -> torch.distributed.run) and
    its timed step (parallel.ShardedStep) at world size 2 over gloo with a fake
    solve: the slabs partition the cube, every rank solves every configuration
    once, and the one all-reduce yields the whole cube's statistics."""
    import json
    import sys
    from pathlib import Path

    sys.path.insert(0, str(Path(__file__).resolve().parent))
    from dist_step_worker import fake_truth

    X, Y, n = 9, 5, 4
    worker = Path(__file__).resolve().parent / "dist_step_worker.py"
    rc = parallel.spawn_ranks(2, [str(worker), str(tmp_path), str(X), str(Y), str(n)],
                              env={"OMP_NUM_THREADS": "1"})
    assert rc == 0
    res = [json.loads((tmp_path / f"rank{r}.json").read_text()) for r in range(2)]
    assert [r["world"] for r in res] == [2, 2]
    slabs = sorted(tuple(r["slab"]) for r in res)
    assert slabs[0][0] == 0 and slabs[-1][1] == X and slabs[0][1] == slabs[1][0]
    assert all(r["solved"] == ["gomp", "cosamp"] for r in res)
    assert all(r["launches"] == 2 * 3 for r in res)     # (2 solver kernels + 1 SSE) x 2 configs
    truth = [fake_truth(p) for p in range(X * Y)]
    ok = [t[2] < 0 for t in truth]
    expect = [float(sum(p * p for p in range(X * Y))),
              sum(1 for t, o in zip(truth, ok) if t[1] and o),
              sum(1 for o in ok if not o),
              sum(1 for t, o in zip(truth, ok) if t[0] == 0 and t[1] and o),
              sum(t[0] for t, o in zip(truth, ok) if o),
              float(sum(range(X * Y)))]
    for r in res:   # every rank holds the reduced statistics, identical for both configs
        for row in r["stats"]:
            np.testing.assert_allclose(row, expect, rtol=1e-12)
