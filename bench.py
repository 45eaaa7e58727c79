#!/usr/bin/env python
"""Benchmark: recovered spectra/s per solver on the B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload scaling|cfg1..cfg4] [--impl ours|reference]

Default workload = BASELINE config 5 (the scaling run the metric is quoted on:
"1/2/4/8 B200"): a 2048 x 868 x 224 synthetic cube (4 x 4 tiles of the
512 x 217 generator, seeds 0..15, 1,777,664 spectra, 90 measured bands per
pixel) recovered by all ten solver configurations (FISTA/ADMM lambda in
{0.1, 100}; gOMP/BIHT/CoSaMP kappa in {27, 33}, G = kappa // 5, mu = 0.1,
eps = 1e-8, caps 5000/2000).  One step = recover the whole cube once with each
configuration (+ PSNR partials + the stats all-reduce).  value = spectra
recovered by all ranks per second (10 x P per step).  Pixel rows are sharded
across ranks (strong scaling of a fixed cube); the only collective is one
NCCL all-reduce of per-configuration PSNR/convergence sums per step.

Inputs come from the frozen generator (paper_2401_14762_b200.synth v1): the
host draws the random stream, the GPU computes spectra, DCT sparsification,
masks and measurements (`--gen host` does it all in numpy); they are
device-resident before timing; the per-step inputs (1.28 GB of measurements)
exceed the 126 MB L2, so no flush is needed.  `--impl reference` times the
CPU oracle (restatement of the reference's solvers; the reference is pure
Python and is not installed on the GPU box) on a bounded pixel sample on all
host cores, rank 0 only.
"""

import argparse
import json
import math
import os
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

from paper_2401_14762_b200 import synth  # noqa: E402

SCALING_SOLVERS = [
    ("fista", dict(lam=0.1), 5000), ("fista", dict(lam=100.0), 5000),
    ("admm", dict(lam=0.1, alpha=1.8), 5000), ("admm", dict(lam=100.0, alpha=1.8), 5000),
    ("gomp", dict(kappa=27, atoms_per_iter=5), None), ("gomp", dict(kappa=33, atoms_per_iter=6), None),
    ("biht", dict(kappa=27, mu=0.1), 2000), ("biht", dict(kappa=33, mu=0.1), 2000),
    ("cosamp", dict(kappa=27), 2000), ("cosamp", dict(kappa=33), 2000),
]
WORKLOADS = {
    "scaling": ("scaling", SCALING_SOLVERS),
    "cfg1": ("jasper", [("gomp", dict(kappa=24, atoms_per_iter=4), None)]),
    "cfg2": ("jasper", [("fista", dict(lam=100.0), 5000), ("admm", dict(lam=100.0, alpha=1.8), 5000)]),
    "cfg3": ("china", [("biht", dict(kappa=22, mu=0.1), 2000), ("gomp", dict(kappa=22, atoms_per_iter=4), None)]),
    "cfg4": ("salinas", [("cosamp", dict(kappa=33), 2000)]),
}
METRIC = "recovered spectra/sec (all solver configs of the workload)"


def label(algo, params):
    return algo + "_" + "_".join(f"{k[0] if k != 'atoms_per_iter' else 'G'}{v:g}" for k, v in params.items()
                                  if k in ("lam", "kappa"))


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


# ------------------------------------------------------------------ CPU oracle leg

CPU_STRIDE = 97


# pixels of the strided sample timed per configuration and step (about 1 s of
# work each on 16 host cores at --ref-budget 1; "all" = the whole sample)
CPU_SAMPLE_PX = {"fista_l0.1": 8192, "admm_l0.1": 1536, "admm_l100": 6144, "cosamp_k27": 6144}


class CpuBaseline:
    """The reference's algorithm on the host cores (the oracle port, one
    worker process per core, OpenBLAS single-threaded per worker, as
    SURVEY.md §8(d) / BASELINE.md §2 prescribe), timed on a fixed
    deterministic sample of the workload cube: every 97th pixel by global
    x-major index (18,327 of the scaling cube's 1,777,664, spread over all 16
    tiles).  Each configuration times a FIXED, evenly spaced subset of that
    sample (CPU_SAMPLE_PX x --ref-budget pixels, else the whole sample), the
    same subset in every step and in both the reference arm and the
    cpu_baseline leg, so the two measure the same work (per-pixel cost is
    heavy-tailed: CoSaMP pixels that cycle to the 2000-iteration cap cost 1000x
    a converging one).  A configuration's rate = subset pixels / wall time of
    its pool map; a step's value = the harmonic aggregate over configurations
    (the way `value` aggregates); also the sum of per-pixel solve times (the
    reference's recovery_time_s semantics, solvers.py:510)."""

    def __init__(self, workload, budget, cores, stride=CPU_STRIDE):
        os.environ["OPENBLAS_NUM_THREADS"] = "1"
        from concurrent.futures import ProcessPoolExecutor
        from oracle import cpu_solvers as oc
        self.oc = oc
        cube_name, self.solvers = WORKLOADS[workload]
        spec = synth.CUBES[cube_name]
        self.shape = [spec["x_dim"], spec["y_dim"], spec["n"]]
        self.sample = synth.generate_strided(cube_name, stride, workers=min(16, cores))
        self.stride, self.budget, self.cores = stride, budget, cores
        self.pool = ProcessPoolExecutor(max_workers=cores, initializer=oc.single_thread_blas)
        list(self.pool.map(abs, range(4 * cores)))        # start the workers outside the timing
        S = self.sample.n_pixels
        self.subset = {}
        for algo, params, _ in self.solvers:
            lab = label(algo, params)
            n = min(S, max(1, int(CPU_SAMPLE_PX.get(lab, S) * budget)))
            self.subset[lab] = (np.arange(n) * S) // n

    def step(self):
        rates, sizes, sum_el = {}, {}, {}
        for algo, params, cap in self.solvers:
            lab = label(algo, params)
            cfg = self.oc.OracleConfig(max_iter=cap or 0, **params)
            idx = self.subset[lab]
            n = len(idx)
            y, masks = np.ascontiguousarray(self.sample.y[idx]), np.ascontiguousarray(self.sample.masks[idx])
            t0 = time.perf_counter()
            # 8 tasks per worker: balances the heavy-tailed configurations without
            # letting the per-task pickling of the basis dominate the cheap ones
            res = self.oc.solve_cube(algo, self.sample.basis, y, masks, cfg,
                                     chunk=max(1, n // (8 * self.cores)), pool=self.pool)
            dt = time.perf_counter() - t0
            rates[lab], sizes[lab], sum_el[lab] = n / dt, n, float(res.elapsed.sum())
        agg = len(rates) / sum(1.0 / r for r in rates.values())
        return agg, rates, sizes, sum_el

    def run(self, warmup, steps):
        vals = []
        for k in range(warmup + steps):
            v = self.step()
            if k >= warmup:
                vals.append(v)
        value = float(np.mean([v[0] for v in vals]))
        labs = list(vals[0][1])
        per = {k: float(np.mean([v[1][k] for v in vals])) for k in labs}
        px = {k: int(sum(v[2][k] for v in vals)) for k in labs}
        sel = {k: float(sum(v[3][k] for v in vals)) for k in labs}
        return {
            "value": value, "unit": "spectra/s", "cores": self.cores, "kind": "port",
            "sample": (f"every {self.stride}th pixel of the {'x'.join(map(str, self.shape))} workload cube "
                       f"(global x-major index p % {self.stride} == 0: {self.sample.n_pixels} px over all tiles); "
                       f"per solver config a fixed evenly spaced subset of it, the same in every step "
                       f"({ {k: len(v) for k, v in self.subset.items()} } px); "
                       f"{steps} timed steps after {warmup} warm-up"),
            "per_solver": per, "pixels_timed": px,
            "sum_elapsed_s": sel,
            "rate_from_sum_elapsed": {k: self.cores * px[k] / sel[k] for k in labs if sel[k] > 0},
        }

    def close(self):
        self.pool.shutdown()


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    cube_name, solvers = WORKLOADS[args.workload]
    spec = synth.CUBES[cube_name]
    cores = host_cores()
    cb = CpuBaseline(args.workload, args.ref_budget, cores)
    try:
        res = cb.run(args.warmup, args.steps)
    finally:
        cb.close()
    value = res["value"]
    P = spec["x_dim"] * spec["y_dim"]
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "spectra/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (generator hcs-synth-v1)",
        "config": {"workload": args.workload, "cube": cube_name, "shape": [spec["x_dim"], spec["y_dim"], spec["n"]],
                   "pixels": P, "measured_bands": synth.measured_count(spec["n"]),
                   "solvers": [label(a, p) for a, p, _ in solvers], "sample": res["sample"]},
        "per_solver": res["per_solver"],
        "cpu_baseline": res,
        "e2e": {"value": value, "unit": "spectra/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ clocks


class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index):
        self.proc = None
        self.path = Path(os.environ.get("TMPDIR", "/tmp")) / f"hcs_clocks_{os.getpid()}.csv"
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={device_index}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except (FileNotFoundError, OSError):
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, smax, reasons = [], [], set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for row in self.path.read_text().splitlines():
            parts = [p.strip() for p in row.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax.append(float(parts[2]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        self.path.unlink(missing_ok=True)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------------ GPU leg


def _ncu_traffic(convex, algo, lab, pixels, n):
    """DRAM bytes (read + write) per launch of the dominant kernel from the
    committed ncu --set full capture of that launch (profiles/), when it
    covers this kernel, configuration and cube size; else None."""
    try:
        rec = json.loads((ROOT / "profiles" / "ncu_traffic_r02.json").read_text())["kernels"]
    except (OSError, ValueError, KeyError):
        return None
    key = (("convex_kernel<%s>" if convex else "greedy_kernel<%s>") % algo) + "|" + lab
    r = rec.get(key)
    if r is None or r.get("pixels") != pixels or r.get("n") != n:
        return None
    return int(r["dram_bytes_read"] + r["dram_bytes_write"])


def _hbm_peak():
    """HBM copy bandwidth of this pool (MEASURED_PEAKS.json, driver-written), else
    the profiling recipe's fallback."""
    try:
        return float(json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs"
    except (OSError, ValueError, KeyError):
        return 6650.0, "of fallback (B200_PROFILING.md, MEASURED_PEAKS.json absent)"


def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2401_14762_b200 import _native, parallel
    from paper_2401_14762_b200.metrics import sse_coeff_partials
    from paper_2401_14762_b200.solvers import SolverConfig, recover_cube, solve_batch
    from paper_2401_14762_b200.transform import Dictionary

    rank, world, local = parallel.dist_env()
    if world > torch.cuda.device_count():
        raise SystemExit(f"bench: {world} ranks but only {torch.cuda.device_count()} visible GPU(s)")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    parallel.init_from_env("nccl", dev)
    _native.load()

    cube_name, solvers = WORKLOADS[args.workload]
    if args.only:
        keep = set(args.only.split(","))
        solvers = [s for s in solvers if label(s[0], s[1]) in keep]
    spec = synth.CUBES[cube_name]
    X = spec["x_dim"]
    x0, x1 = parallel.row_slab(X, rank, world)
    torch.cuda.synchronize()
    t_gen = time.perf_counter()
    if args.gen == "device":
        # input side on the GPU (hcs_synth_spectra + hcs_sparsify_measure; host draws the random stream)
        cube = synth.generate_named_device(cube_name, x_range=(x0, x1), device=dev, with_coeffs=True)
        y_d, masks_d, spectra_d, coeffs_d = cube.y, cube.masks, cube.spectra, cube.coeffs
    else:
        cube = synth.generate_named(cube_name, x_range=(x0, x1), workers=min(16, host_cores()))
        y_d = torch.as_tensor(cube.y, device=dev)
        masks_d = torch.as_tensor(cube.masks, device=dev)
        spectra_d = torch.as_tensor(cube.spectra, device=dev)
        coeffs_d = torch.as_tensor(cube.coeffs, device=dev)
    torch.cuda.synchronize()
    t_gen = time.perf_counter() - t_gen
    P, n, m = cube.n_pixels, cube.n, cube.m
    P_total = X * spec["y_dim"]
    basis_d = torch.as_tensor(cube.basis, device=dev)
    # timed input-side pass (device-resident spectra and keys): HBM + DMMA throughput of
    # hcs_sparsify_measure over this rank's slab, reported beside the solvers
    input_side = None
    if args.gen == "device":
        from paper_2401_14762_b200 import sparsify as sp
        kg = torch.Generator(device=dev).manual_seed(1234)
        keys_d = torch.rand((P, n), dtype=torch.float64, device=dev, generator=kg)
        sp.sparsify_measure(spectra_d, basis_d, m, rule="maxrel", factor=synth.SPARSIFY_T, keys=keys_d,
                            with_coeffs=False)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3):
            sp.sparsify_measure(spectra_d, basis_d, m, rule="maxrel", factor=synth.SPARSIFY_T, keys=keys_d,
                                with_coeffs=False)
        e1.record()
        torch.cuda.synchronize()
        t_in = e0.elapsed_time(e1) / 3e3
        nbytes = P * (8 * n + 8 * n + 8 * n + 8 * m + m)     # spectra + keys in; spectra, y, masks out
        input_side = {"kernel": "sparsify_measure_kernel", "pixels": P, "ms": 1e3 * t_in,
                      "spectra_per_s": P / t_in, "hbm_gbps": nbytes / t_in / 1e9,
                      "dmma_tflops": 4.0 * n * n * P / t_in / 1e12,
                      "note": "c = Psi^T f, T max|c| threshold, f_s = Psi c, M smallest keys, y = f_s[mask]; "
                              "4 N^2 FLOP and 24N + 9M bytes per spectrum"}
        del keys_d
    cfgs = [(a, p, SolverConfig(time_limit=None, max_iter=cap, **p)) for a, p, cap in solvers]
    nsolv = len(cfgs)
    # PSNR peak = max |reference spectra| over the whole cube: input-derived, reduced once at setup
    peak_ref = float(parallel.all_reduce_max(spectra_d.abs().max().reshape(1)).item())
    # the timed step: every configuration on this rank's slab + PSNR partials + one all-reduce
    step = parallel.ShardedStep([(a, c) for a, _, c in cfgs], y_d, masks_d, basis_d, coeffs_d)
    stats_d = step.stats
    torch.cuda.synchronize()

    # FP64 tensor peak of this GPU (roofline denominator)
    peak_tf = _native.dmma_peak_tflops()

    print(f"[bench] rank {rank}: {P} px generated in {t_gen:.1f}s; dmma peak {peak_tf:.1f} TF/s", file=sys.stderr,
          flush=True)
    for _ in range(args.warmup):
        tw = time.perf_counter()
        step()
        torch.cuda.synchronize()
        print(f"[bench] warm-up step {time.perf_counter() - tw:.2f}s", file=sys.stderr, flush=True)
    torch.cuda.synchronize()
    step.check_errors()

    ev = [[[torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)] for _ in cfgs]
          for _ in range(args.steps)]
    clocks = ClockSampler(local)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record()
    for k in range(args.steps):
        step(ev[k])
    t1.record()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    step.check_errors()
    out = step.out
    elapsed = t0.elapsed_time(t1) / 1e3
    per_cfg = np.array([[ev[k][i][0].elapsed_time(ev[k][i][1]) / 1e3 for i in range(nsolv)]
                        for k in range(args.steps)]).mean(axis=0)
    tt = torch.tensor([elapsed, *per_cfg], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    elapsed = float(tt[0])
    per_cfg = tt[1:].cpu().numpy()
    stats = stats_d.cpu().numpy()

    # roofline of the dominant kernel: the configuration with the longest launch
    # (events around its hcs_recover call inside the timed region, max over ranks)
    dom = int(np.argmax(per_cfg))
    d_algo, d_params, _ = cfgs[dom]
    convex = d_algo in ("fista", "admm")
    work_all = float(stats[dom, 5])                 # algorithmic FLOPs of that launch, all ranks
    achieved = work_all / per_cfg[dom] / world / 1e12
    roofline = {"bound": "tensor", "unit": "TFLOP/s", "achieved": achieved, "peak": peak_tf,
                "frac": achieved / peak_tf, "traffic": _ncu_traffic(convex, d_algo, label(d_algo, d_params), P_total, n),
                "kernel": ("convex_kernel<%s>" if convex else "greedy_kernel<%s>") % d_algo,
                "config": label(d_algo, d_params), "launch_ms": 1e3 * per_cfg[dom],
                "peak_source": "FP64 DMMA m8n8k4 throughput measured on this GPU by hcs_dmma_peak_tflops "
                               "(MEASURED_PEAKS.json has no FP64 figure)",
                "algorithmic": ("4 N^2 FLOP per pixel-iteration (two N x N FP64 GEMMs)" if convex else
                                "per pass 2NM (correlation) + LS(M,k) = 2Mk^2 - 2k^3/3 + 4Mk - k^2 per "
                                "least-squares solve + 2Mk (residual), k from the actual supports")
                               + f"; N={n}, M={m}; {work_all:.4g} FLOP in the launch (all ranks), per GPU",
                "per_config_tflops": {label(a, p): float(stats[i, 5]) / per_cfg[i] / world / 1e12
                                      for i, (a, p, _) in enumerate(cfgs)},
                "per_config_frac": {label(a, p): float(stats[i, 5]) / per_cfg[i] / world / 1e12 / peak_tf
                                    for i, (a, p, _) in enumerate(cfgs)},
                "work_note": "device work counters: 4 N^2 per slot-engine iteration (the algorithmic count; "
                             "FISTA's second GEMM skips all-zero k-steps when at most half are active, counted "
                             "dense), 12 N per iteration of the certified zero-shrinkage ADMM pass (admm_l100, "
                             "the FLOPs it executes), greedy per-pass counts from the actual supports"}

    # streaming phase: the coefficient-domain PSNR kernel alone (HBM-bound), timed
    # with events on its stream over the last recovered cube
    sse_tmp = torch.zeros(1, dtype=torch.float64, device=dev)
    sse_coeff_partials(coeffs_d, out.x, out=sse_tmp)
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s0.record()
    for _ in range(10):
        sse_coeff_partials(coeffs_d, out.x, out=sse_tmp)
    s1.record()
    torch.cuda.synchronize()
    t_sse = s0.elapsed_time(s1) / 10e3
    hbm_peak, hbm_src = _hbm_peak()
    sse_bytes = 2 * 8 * P * n
    streaming = {"bound": "hbm", "kernel": "sse_coeff_kernel", "unit": "GB/s", "achieved": sse_bytes / t_sse / 1e9,
                 "peak": hbm_peak, "frac": sse_bytes / t_sse / 1e9 / hbm_peak, "launch_ms": 1e3 * t_sse,
                 "peak_source": hbm_src,
                 "algorithmic": f"16 bytes per voxel (reference + recovered coefficient), {P} x {n} voxels per rank; "
                                "PSNR squared error by Parseval, no spectra GEMM"}

    total_spectra = P_total * nsolv * args.steps
    value = total_spectra / elapsed
    per_solver = {label(a, p): P_total / t for (a, p, _), t in zip(cfgs, per_cfg)}
    quality = {label(a, p): parallel.cube_summary(stats[i], peak_ref, P_total, n)
               for i, (a, p, _) in enumerate(cfgs)}

    # ---- end to end through the public API, host (pinned) buffers ----------------
    e2e = None
    if not args.no_e2e:
        y_host = cube.y.cpu().numpy() if isinstance(cube.y, torch.Tensor) else cube.y
        masks_host = cube.masks.cpu().numpy() if isinstance(cube.masks, torch.Tensor) else cube.masks
        y_h = torch.from_numpy(y_host.reshape(x1 - x0, spec["y_dim"], m)).pin_memory()
        dic = Dictionary.per_pixel(cube.basis, masks_host)
        # two reusable pinned output cubes (pinning 3 GB per call would cost ~1.6 s; a
        # pipeline over many cubes keeps its output buffers)
        outs = [torch.empty((x1 - x0, spec["y_dim"], n), dtype=torch.float64, pin_memory=True) for _ in range(2)]
        h2d = d2h = 0
        print(f"[bench] e2e warm-up", file=sys.stderr, flush=True)
        for _ in range(1):   # warm-up of the e2e path
            recover_cube(y_h, dic, cfgs[-1][2], cfgs[-1][0], out=outs[0])
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        te = time.perf_counter()
        for k in range(args.e2e_steps):
            for i, (algo, _, cfg) in enumerate(cfgs):
                cube_h, st = recover_cube(y_h, dic, cfg, algo, out=outs[i % 2])
                if k == 0:
                    h2d += y_h.numel() * 8 + masks_host.size
                    # the cube, plus the five aggregate statistics reduced on the device
                    # (per-pixel stats arrays are copied only when read)
                    d2h += cube_h.numel() * 8 + 5 * 8
        torch.cuda.synchronize()
        te = time.perf_counter() - te
        tte = torch.tensor([te], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(tte, op=dist.ReduceOp.MAX)
        te = float(tte[0])
        e2e = {"value": P_total * nsolv * args.e2e_steps / te, "unit": "spectra/s",
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
               "api": "paper_2401_14762_b200.recover_cube (pinned host measurements, per-pixel Dictionary, pinned out= cube; chunked H2D/solve/D2H pipeline)",
               "steps": args.e2e_steps}

    # ---- CPU baseline (rank 0, N = 1 only) --------------------------------------------
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cb = CpuBaseline(args.workload, args.ref_budget, host_cores())
        try:
            cpu = cb.run(1, 2)
        finally:
            cb.close()

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "spectra/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * elapsed / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (generator hcs-synth-v1; " + ("input side generated on the GPU from the host-drawn "
                    "random stream" if args.gen == "device" else "host-generated") + ", device-resident before timing)",
            "config": {"workload": args.workload, "cube": cube_name, "shape": [X, spec["y_dim"], n],
                       "pixels": P_total, "measured_bands": m, "solvers": [label(a, p) for a, p, _ in cfgs],
                       "parallelism": f"pixel-row slabs x{world}", "l2": "inputs (1.28 GB/step) > 126 MB L2; no flush"},
            "per_solver": per_solver, "quality": quality,
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": step.launches * args.steps,
            "clocks": clk, "generation_s": t_gen, "input_side": input_side, "streaming": streaming,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default="scaling", choices=sorted(WORKLOADS))
    ap.add_argument("--impl", default="ours", choices=("ours", "reference"))
    ap.add_argument("--e2e-steps", type=int, default=1)
    ap.add_argument("--ref-budget", type=float, default=1.0,
                    help="scale of the CPU sample per solver config (1: ~1 s of work per config and step on 16 "
                         "cores; reference arm and the cpu_baseline leg)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--only", default="", help="comma-separated solver labels (diagnostics)")
    ap.add_argument("--gen", default="device", choices=("device", "host"),
                    help="where the cube's input side is computed (same cube up to FP64 rounding)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: re-launch this command as N ranks (torch.distributed.run, 127.0.0.1)
        from paper_2401_14762_b200 import parallel
        return parallel.spawn_ranks(args.gpus, [str(Path(__file__).resolve()), *sys.argv[1:]])
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
