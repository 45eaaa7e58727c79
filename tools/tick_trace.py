"""Per-warp timeline of the convex engine's ticks (HCS_TRACE build):
    HCS_LIB=variants/libtrace.so python tools/tick_trace.py --algo admm
marks: 0 tick start, 1 slot phase done, 2 GEMM 1 done, 3 barrier out, 4 epilogue 1 done, 5 barrier out,
6 GEMM 2 done, 7 (fista) barrier out, 8 epilogue 2 done, 9 barrier out.  Cycles relative to the tick start of warp 0."""
import argparse, ctypes, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
from paper_2401_14762_b200 import _native, synth
from paper_2401_14762_b200.solvers import SolverConfig, solve_batch
ap = argparse.ArgumentParser(); ap.add_argument("--algo", default="admm"); a = ap.parse_args()
c = synth.generate(400, 100, 224, seed=11)
dev = torch.device("cuda")
solve_batch(a.algo, torch.as_tensor(c.y, device=dev), torch.as_tensor(c.masks, device=dev), torch.as_tensor(c.basis, device=dev),
            SolverConfig(lam=0.1, time_limit=None, max_iter=5000))
torch.cuda.synchronize()
buf = (ctypes.c_longlong * 768)()
assert _native.load().hcs_debug_trace_cx(buf) == 0
t = np.array(buf[:]).reshape(4, 16, 12)
names = ["start", "slots", "gemm1", "bar", "epi1", "bar", "gemm2", "bar", "epi2", "bar"]
for k in range(1, 3):
    base = t[k, 0, 0]
    print(f"tick {200 + k}: length {t[k + 1, 0, 0] - base} cycles; per warp, cycles since the tick start of warp 0")
    print("warp " + " ".join(f"{n:>7}" for n in names))
    for w in range(16):
        print(f"{w:4d} " + " ".join(f"{int(t[k, w, m] - base):7d}" for m in range(10)))
