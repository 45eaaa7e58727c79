"""Rank process for tests/test_distributed.py: launched by
paper_2401_14762_b200.parallel.spawn_ranks (torch.distributed.run, the same
launcher `bench.py --gpus N` uses), it runs parallel.ShardedStep -- the
bench's timed step -- over gloo on CPU with a fake solve hook, and writes
its slab and the reduced statistics to <out>/rank<r>.json.

    python tests/dist_step_worker.py <out_dir> <X> <Y> <n>
"""

import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

from paper_2401_14762_b200 import parallel  # noqa: E402


def fake_truth(p):
    """Deterministic per-pixel outcome of global pixel p (a stand-in solver)."""
    it = p % 7
    conv = p % 3 != 0
    failed = 2 if p % 11 == 0 else -1
    return it, conv, failed, float(p)


class FakeBatch:
    def __init__(self, gidx, n):
        vals = [fake_truth(int(p)) for p in gidx]
        self.x = torch.zeros((len(gidx), n), dtype=torch.float64)
        self.iterations = torch.tensor([v[0] for v in vals], dtype=torch.int32)
        self.converged = torch.tensor([v[1] for v in vals], dtype=torch.uint8)
        self.failed_at = torch.tensor([v[2] for v in vals], dtype=torch.int32)
        self.work = torch.tensor([v[3] for v in vals], dtype=torch.float64)
        self.launches = 2

    def error_flag(self):
        return torch.zeros((1,), dtype=torch.int32)


def main():
    out, X, Y, n = Path(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
    rank, world, _ = parallel.init_from_env("gloo")
    x0, x1 = parallel.row_slab(X, rank, world)
    gidx = torch.arange(x0 * Y, x1 * Y, dtype=torch.int64)
    P = len(gidx)
    y = torch.zeros((P, 3), dtype=torch.float64)
    masks = torch.zeros((P, 3), dtype=torch.uint8)
    basis = torch.eye(n, dtype=torch.float64)
    # reference coefficients: pixel p's row is (p, 0, ...), so its SSE against x = 0 is p^2
    coeffs = torch.zeros((P, n), dtype=torch.float64)
    coeffs[:, 0] = gidx.to(torch.float64)
    seen = []

    def solve(algo, y_, m_, b_, cfg, out=None):
        seen.append(algo)
        return FakeBatch(gidx.tolist(), n)

    def sse(ref, x, out=None):
        out += ((ref - x) ** 2).sum()

    step = parallel.ShardedStep([("gomp", None), ("cosamp", None)], y, masks, basis, coeffs, solve=solve, sse=sse)
    launches = step()
    step.check_errors()
    (out / f"rank{rank}.json").write_text(json.dumps({
        "rank": rank, "world": world, "slab": [x0, x1], "stats": step.stats.tolist(), "launches": launches,
        "solved": seen}))
    import torch.distributed as dist
    if dist.is_initialized():
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
