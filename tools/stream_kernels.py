"""Throughput of the streaming kernels on scaling-cube-sized arrays (1,777,664 x 224):
hcs_psnr_partials and hcs_sparsify_measure (keys -> masks), CUDA events, best of 5."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2401_14762_b200 import synth, sparsify as sp
from paper_2401_14762_b200.metrics import psnr_partials

P, n, m = 1777664, 224, 90
dev = torch.device("cuda")
g = torch.Generator(device=dev).manual_seed(0)
f = torch.rand((P, n), dtype=torch.float64, device=dev, generator=g)
keys = torch.rand((P, n), dtype=torch.float64, device=dev, generator=g)
x = torch.rand((P, n), dtype=torch.float64, device=dev, generator=g)
b = torch.as_tensor(synth.dct_basis(n), device=dev)
out = torch.zeros(2, dtype=torch.float64, device=dev)


def best(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    t = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        t.append(e0.elapsed_time(e1) / 1e3)
    return min(t)


t = best(lambda: psnr_partials(f, x, b, out=out))
print(f"psnr_partials: {1e3 * t:.2f} ms, {16 * n * P / t / 1e9:.0f} GB/s (16N B/px), {2 * n * n * P / t / 1e12:.1f} TF/s")
t = best(lambda: sp.sparsify_measure(f, b, m, rule="maxrel", factor=0.1, keys=keys, with_coeffs=False))
print(f"sparsify_measure: {1e3 * t:.2f} ms, {P * (24 * n + 9 * m) / t / 1e9:.0f} GB/s (24N+9M B/px), "
      f"{4 * n * n * P / t / 1e12:.1f} TF/s")
