"""Position-sensitive digests of every output of the convex configurations on the full bench cube
(2048 x 868 x 224, 1,777,664 pixels), for a bit-for-bit comparison of two library builds:

    HCS_LIB=variants/libhead.so python tools/cube_digest.py > a.json
    python tools/cube_digest.py > b.json;  python tools/cube_digest.py --compare a.json b.json

Digest of an array = (wrap-around int64 sum of its bit pattern, wrap-around sum of bit pattern x
(2 index + 1)), computed on the GPU; iterations / converged / failed_at additionally by plain sums."""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def digest(t):
    import torch
    v = t.contiguous().view(-1)
    if v.dtype == torch.float64:
        v = v.view(torch.int64)
    else:
        v = v.to(torch.int64)
    w = torch.arange(v.numel(), device=v.device, dtype=torch.int64) * 2 + 1
    return [int(v.sum().item()), int((v * w).sum().item())]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--compare", nargs=2)
    ap.add_argument("--cube", default="scaling")
    args = ap.parse_args()
    if args.compare:
        a, b = (json.loads(Path(p).read_text()) for p in args.compare)
        ok = True
        for k in a["configs"]:
            same = a["configs"][k] == b["configs"].get(k)
            ok &= same
            print(f"{k}: bit-for-bit identical outputs over {a['pixels']} pixels: {same}")
        print(f"libraries: {a['lib']}  vs  {b['lib']}")
        sys.exit(0 if ok else 1)
    import os
    import torch
    from paper_2401_14762_b200 import _native, synth
    from paper_2401_14762_b200.solvers import SolverConfig, solve_batch
    dev = torch.device("cuda")
    cube = synth.generate_named_device(args.cube, device=dev, with_coeffs=False)
    basis = torch.as_tensor(cube.basis, device=dev)
    out = {"lib": os.environ.get("HCS_LIB", str(_native.LIB_PATH)), "pixels": int(cube.y.shape[0]), "configs": {}}
    for algo, lam in (("fista", 0.1), ("fista", 100.0), ("admm", 0.1), ("admm", 100.0)):
        b = solve_batch(algo, cube.y, cube.masks, basis, SolverConfig(lam=lam, time_limit=None, max_iter=5000))
        torch.cuda.synchronize()
        out["configs"][f"{algo}_l{lam:g}"] = {
            "x": digest(b.x), "iterations": digest(b.iterations), "converged": digest(b.converged),
            "final_delta": digest(b.final_delta), "failed_at": digest(b.failed_at),
            "admm_gap": digest(b.admm_gap) if b.admm_gap is not None else None,
            "total_iterations": int(b.iterations.sum().item()), "n_converged": int(b.converged.sum().item())}
        del b
    print(json.dumps(out))


if __name__ == "__main__":
    main()
