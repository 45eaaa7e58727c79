import sys, time
sys.path.insert(0, '/root/repo')
import numpy as np, torch
from paper_2401_14762_b200 import synth
from paper_2401_14762_b200.solvers import SolverConfig, recover_cube, solve_batch
from paper_2401_14762_b200.transform import Dictionary
import bench
dev = torch.device('cuda')
c = synth.generate_named_device('scaling', device=dev)
X, Y = c.shape; n, m = c.n, c.m
y_h = torch.from_numpy(c.y.cpu().numpy().reshape(X, Y, m)).pin_memory()
dic = Dictionary.per_pixel(c.basis, c.masks.cpu().numpy())
out = torch.empty((X, Y, n), dtype=torch.float64, pin_memory=True)
basis_d = torch.as_tensor(c.basis, device=dev)
for algo, params, cap in bench.SCALING_SOLVERS:
    cfg = SolverConfig(time_limit=None, max_iter=cap, **params)
    recover_cube(y_h, dic, cfg, algo, out=out)
    torch.cuda.synchronize()
    t = time.perf_counter(); recover_cube(y_h, dic, cfg, algo, out=out); torch.cuda.synchronize(); te = time.perf_counter() - t
    b = solve_batch(algo, c.y, c.masks, basis_d, cfg); torch.cuda.synchronize()
    t = time.perf_counter(); b = solve_batch(algo, c.y, c.masks, basis_d, cfg, out=b); torch.cuda.synchronize(); td = time.perf_counter() - t
    for ch in (111104, 444416):
        t = time.perf_counter(); recover_cube(y_h, dic, cfg, algo, out=out, chunk_pixels=ch); torch.cuda.synchronize(); tc = time.perf_counter() - t
        print(f"   chunk {ch}: {tc*1e3:.1f} ms")
    print(f"{bench.label(algo, params):12s} e2e {te*1e3:8.1f} ms  device {td*1e3:8.1f} ms  overhead {1e3*(te-td):7.1f} ms", flush=True)
