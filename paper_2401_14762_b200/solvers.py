"""Per-pixel sparse recovery solvers on the B200: the reference's solver API.

Drop-in for `hypercs.solvers` (`/root/reference/pkg/src/hypercs/solvers.py`):
`SolverConfig` (:40-85), `SolverResult` (:88-95), `StopDecision`/`stop_check`
(:98-127), `lasso_objective` (:130-134), the five solvers and `SOLVERS`
(:164-405), `NumericalFailure` (:32-37), `RecoveryStats` (:413-433),
`derive_pixel_seed` (:408-410) and `recover_cube` (:455-514).

Every solve runs in libhypercs_b200.so (hand-written sm_100a kernels); this
module validates, moves arrays and assembles results.  Differences from the
reference:

* real FP64 throughout; the recovered cube is float64 (the reference's is
  complex128 with identically zero imaginary part for real bases);
* per-pixel masks are supported (`Dictionary.per_pixel`);
* `time_limit` is a per-pixel device-clock budget measured from the moment a
  pixel enters the solver; `elapsed` is that pixel's device time.  With a
  budget set (the default is 2 s, as in the reference) a gOMP / CoSaMP pixel
  whose iterates cycle runs until the budget or `max_iter` expires, like the
  reference's; with `time_limit=None` the kernel detects the exact state cycle
  and jumps to the iteration cap's result (same output, `hcs_greedy.cu`), so
  batch runs over cycling cubes (CoSaMP kappa = 33) should pass None;
* `jobs` is accepted and ignored: pixels are scheduled by the GPU's work queue
  (multi-GPU sharding lives in `paper_2401_14762_b200.parallel`).
"""

import enum
import math
from dataclasses import dataclass, field

import numpy as np

from . import _native as nat
from .transform import Dictionary


class NumericalFailure(RuntimeError):
    """A solver produced non-finite values; iteration stores where."""

    def __init__(self, iteration):
        super().__init__(f"non-finite values at iteration {iteration}")
        self.iteration = iteration


@dataclass
class SolverConfig:
    """Shared solver parameters, validated exactly as solvers.py:67-85."""

    lam: float = 0.1
    kappa: int = 1
    atoms_per_iter: int | None = None
    mu: float = 0.1
    alpha: float = 1.8
    epsilon: float = 1e-8
    time_limit: float | None = 2.0
    max_iter: int | None = None
    seed: int = 0

    def __post_init__(self):
        if self.lam < 0:
            raise ValueError("lam must be >= 0")
        if self.kappa < 1:
            raise ValueError("kappa must be >= 1")
        if self.atoms_per_iter is None:
            self.atoms_per_iter = max(1, self.kappa // 5)
        if not 1 <= self.atoms_per_iter <= self.kappa:
            raise ValueError("atoms_per_iter must be in [1, kappa]")
        if self.mu <= 0:
            raise ValueError("mu must be > 0")
        if self.alpha <= 0:
            raise ValueError("alpha must be > 0")
        if self.epsilon <= 0:
            raise ValueError("epsilon must be > 0")
        if self.time_limit is not None and self.time_limit <= 0:
            raise ValueError("time_limit must be > 0 or None")
        if self.max_iter is not None and self.max_iter < 1:
            raise ValueError("max_iter must be >= 1 or None")

    def to_native(self):
        if self.max_iter is not None and self.max_iter > 2**31 - 1:
            raise ValueError("max_iter must fit in int32")
        return nat.HcsParams(
            lam=float(self.lam), mu=float(self.mu), alpha=float(self.alpha), epsilon=float(self.epsilon),
            kappa=int(self.kappa), atoms_per_iter=int(self.atoms_per_iter),
            max_iter=int(self.max_iter or 0), reserved=0,
            time_limit=float(self.time_limit) if self.time_limit is not None else 0.0)


@dataclass
class SolverResult:
    x: np.ndarray
    iterations: int
    converged: bool
    elapsed: float
    final_delta: float
    admm_gap: float | None = None  # ||x - z|| at termination, admm only


class StopDecision(enum.Enum):
    CONTINUE = "continue"
    CONVERGED = "converged"
    TIMEOUT = "timeout"
    ITER_CAP = "iter_cap"


@dataclass
class SolverState:
    """Residual bookkeeping consulted by the stop rule (solvers.py:105-112)."""

    residual: np.ndarray
    residual_prev: np.ndarray | None = None
    delta: float = 1.0
    iterations: int = 0


def stop_check(state, config, elapsed):
    """The stop rule every device solver applies before each pass
    (solvers.py:115-127): converged > timeout > iteration cap."""
    if state.delta < config.epsilon:
        return StopDecision.CONVERGED
    if config.time_limit is not None and elapsed >= config.time_limit:
        return StopDecision.TIMEOUT
    if config.max_iter is not None and state.iterations >= config.max_iter:
        return StopDecision.ITER_CAP
    return StopDecision.CONTINUE


def lasso_objective(x, y, dictionary, lam):
    """H(x) = 0.5 ||A x - y||^2 + lam * sum |x_i| (solvers.py:130-134)."""
    matrix = dictionary.matrix if hasattr(dictionary, "matrix") else np.asarray(dictionary)
    r = matrix @ x - y
    return 0.5 * float(np.real(np.vdot(r, r))) + lam * float(np.abs(x).sum())


SOLVER_NAMES = ("fista", "admm", "gomp", "biht", "cosamp")
CONVEX_SOLVERS = ("fista", "admm")
GREEDY_SOLVERS = ("gomp", "biht", "cosamp")


def derive_pixel_seed(run_seed, pixel_index):
    """Stable per-pixel seed (solvers.py:408-410); kept for API parity."""
    return (run_seed * 6364136223846793005 + pixel_index * 1442695040888963407) % (2**63)


# ----------------------------------------------------------------- device batch


@dataclass
class DeviceBatch:
    """Raw device outputs of one hcs_recover call (CUDA tensors)."""

    x: object            # (P, n) float64
    iterations: object   # (P,) int32
    converged: object    # (P,) uint8
    final_delta: object  # (P,) float64
    failed_at: object    # (P,) int32
    admm_gap: object     # (P,) float64
    lipschitz: object    # (P,) float64
    elapsed: object      # (P,) float64
    work: object = None  # (P,) float64 algorithmic FLOPs executed
    trace: object = None
    trace_len: object = None
    workspace: object = None
    launches: int = 0        # kernels this call launched (prep + solver)
    algorithm: str = ""

    def error_flag(self):
        """The device word hcs_recover_status reads (int32 view into the
        workspace; non-zero after a non-finite measurement)."""
        return self.workspace[8:12].view(__import__("torch").int32)

    def check_status(self, stream=None):
        """Raise ValueError where the reference raises on non-finite input (syncs)."""
        nat.check(nat.load().hcs_recover_status(nat.ptr(self.workspace), nat.stream_handle(stream)))


def solve_batch(algorithm, y, masks, basis, config, trace_calls=0, stream=None, workspace=None,
                check_status=True, out=None):
    """One hcs_recover call on device tensors: y (P, m) float64, masks (P, m)
    uint8, basis (n, n) float64, all CUDA.  Returns a DeviceBatch; raises
    ValueError exactly where the reference raises (config, preconditions,
    non-finite measurements for admm/gomp/biht/cosamp).  With
    check_status=False the call is fully asynchronous and the caller runs
    ``batch.check_status()`` later.  ``out`` (a DeviceBatch of the same
    algorithm and shape) reuses its buffers instead of allocating."""
    import torch
    if algorithm not in nat.ALGO_IDS:
        raise ValueError(f"unknown algorithm {algorithm!r}")
    lib = nat.load()
    P, m = int(y.shape[0]), int(y.shape[1])
    n = int(basis.shape[0])
    dev = y.device
    f64 = dict(dtype=torch.float64, device=dev)
    if out is not None and tuple(out.x.shape) == (P, n) and trace_calls == 0:
        workspace = out.workspace if workspace is None else workspace
        if out.algorithm != algorithm:
            # fields only some solvers write (admm_gap: admm; lipschitz: fista)
            out.admm_gap.fill_(math.nan)
            out.lipschitz.fill_(math.nan)
    else:
        out = None
    out = out or DeviceBatch(
        x=torch.empty((P, n), **f64),
        iterations=torch.empty((P,), dtype=torch.int32, device=dev),
        converged=torch.empty((P,), dtype=torch.uint8, device=dev),
        final_delta=torch.empty((P,), **f64),
        failed_at=torch.empty((P,), dtype=torch.int32, device=dev),
        admm_gap=torch.full((P,), math.nan, **f64),
        lipschitz=torch.full((P,), math.nan, **f64),
        elapsed=torch.empty((P,), **f64),
        work=torch.empty((P,), **f64),
    )
    st = nat.HcsStats(iterations=out.iterations.data_ptr(), converged=out.converged.data_ptr(),
                      final_delta=out.final_delta.data_ptr(), failed_at=out.failed_at.data_ptr(),
                      admm_gap=out.admm_gap.data_ptr(), lipschitz=out.lipschitz.data_ptr(),
                      elapsed=out.elapsed.data_ptr(), work=out.work.data_ptr(), trace=None, trace_len=None,
                      trace_calls=0)
    if trace_calls > 0:
        out.trace = torch.zeros((P, trace_calls, 4), dtype=torch.int64, device=dev)
        out.trace_len = torch.zeros((P,), dtype=torch.int32, device=dev)
        st.trace = out.trace.data_ptr()
        st.trace_len = out.trace_len.data_ptr()
        st.trace_calls = trace_calls
    algo = nat.ALGO_IDS[algorithm]
    wsb = lib.hcs_workspace_bytes(algo, P, n, m)
    if workspace is None or workspace.numel() < wsb:
        workspace = torch.empty((max(wsb, 256),), dtype=torch.uint8, device=dev)
    prm = config.to_native()
    sh = nat.stream_handle(stream)
    nat.check(lib.hcs_recover(algo, P, n, m, nat.ptr(basis), nat.ptr(y), nat.ptr(masks), prm, nat.ptr(out.x),
                              st, nat.ptr(workspace), workspace.numel(), sh))
    out.workspace = workspace
    out.algorithm = algorithm
    out.launches = lib.hcs_recover_launches(algo, n, m, prm) if P > 0 else 0
    if check_status:
        out.check_status(stream)
    return out


# ----------------------------------------------------------------- per pixel


def _one_pixel(algorithm, y, dictionary, config):
    import torch
    if not isinstance(dictionary, Dictionary):
        dictionary = Dictionary.from_matrix(dictionary.matrix if hasattr(dictionary, "matrix") else dictionary)
    if not dictionary.shared:
        raise ValueError("per-pixel solvers take a single-mask dictionary")
    y = np.asarray(y)
    if np.iscomplexobj(y):
        if np.any(y.imag != 0):
            raise ValueError("the GPU backend is real-valued")
        y = y.real
    y = np.asarray(y, dtype=np.float64)
    if y.shape != (dictionary.m,):
        raise ValueError(f"measurement length {y.shape} does not match {dictionary.m} rows")
    basis_d, masks_d = dictionary.device_arrays("cuda", 1)
    yd = torch.as_tensor(y, device="cuda").reshape(1, -1)
    b = solve_batch(algorithm, yd, masks_d, basis_d, config)
    failed = int(b.failed_at[0].item())
    if failed >= 0:
        raise NumericalFailure(failed)
    gap = float(b.admm_gap[0].item()) if algorithm == "admm" else None
    if gap is not None and math.isnan(gap):
        gap = None
    return SolverResult(
        x=b.x[0].cpu().numpy(), iterations=int(b.iterations[0].item()), converged=bool(b.converged[0].item()),
        elapsed=float(b.elapsed[0].item()), final_delta=float(b.final_delta[0].item()), admm_gap=gap)


def fista(y, dictionary, config):
    """Accelerated proximal-gradient lasso solve (solvers.py:164-203), on the GPU."""
    return _one_pixel("fista", y, dictionary, config)


def admm(y, dictionary, config):
    """Scaled-dual ADMM lasso solve returning z (solvers.py:206-245), on the GPU."""
    return _one_pixel("admm", y, dictionary, config)


def gomp(y, dictionary, config):
    """Generalized OMP with a kappa-prune re-solve (solvers.py:248-297), on the GPU."""
    return _one_pixel("gomp", y, dictionary, config)


def biht(y, dictionary, config):
    """Hard thresholding with a least-squares prune (solvers.py:300-342), on the GPU."""
    return _one_pixel("biht", y, dictionary, config)


def cosamp(y, dictionary, config):
    """Compressive sampling matching pursuit (solvers.py:345-394), on the GPU."""
    return _one_pixel("cosamp", y, dictionary, config)


SOLVERS = {"fista": fista, "admm": admm, "gomp": gomp, "biht": biht, "cosamp": cosamp}


# ----------------------------------------------------------------- whole cubes


class _LazyResults:
    """RecoveryStats.results without building P Python objects up front."""

    def __init__(self, stats, x):
        self._s, self._x = stats, x

    def __len__(self):
        return self._s.n_pixels

    def __getitem__(self, i):
        if isinstance(i, slice):
            return [self[j] for j in range(*i.indices(len(self)))]
        s = self._s
        if s.failed_at[i] >= 0:
            return None
        gap = None
        if s.algorithm == "admm" and not math.isnan(s.admm_gap[i]):
            gap = float(s.admm_gap[i])
        x = self._x[i]
        x = x.cpu().numpy() if hasattr(x, "cpu") else np.asarray(x)
        return SolverResult(x=x, iterations=int(s.iterations[i]), converged=bool(s.converged[i]),
                            elapsed=float(s.elapsed[i]), final_delta=float(s.final_delta[i]), admm_gap=gap)

    def __iter__(self):
        return (self[i] for i in range(len(self)))


_PER_PIXEL = ("iterations", "converged", "final_delta", "failed_at", "admm_gap", "elapsed")


@dataclass
class RecoveryStats:
    """Aggregate of a whole-cube recovery (solvers.py:413-433), plus the
    per-pixel arrays the GPU produces (host numpy: `iterations`, `converged`,
    `final_delta`, `failed_at`, `admm_gap`, `elapsed`).  The aggregates are
    reduced on the device; the per-pixel arrays are copied to the host on
    first access (most callers only read the aggregates)."""

    n_pixels: int
    n_converged: int
    n_failed: int
    n_zero_pixels: int
    total_iterations: int
    recovery_time_s: float
    results: object = field(repr=False, default=None)
    failed_pixels: list = field(default_factory=list)
    algorithm: str = ""
    wall_time_s: float = 0.0
    _src: dict = field(repr=False, default_factory=dict)     # name -> device tensor (until first access)
    _host: dict = field(repr=False, default_factory=dict)    # name -> numpy array

    def _array(self, name):
        a = self._host.get(name)
        if a is None:
            t = self._src.pop(name)
            a = t.cpu().numpy()
            if name == "converged":
                a = a.astype(bool)
            self._host[name] = a
        return a

    iterations = property(lambda self: self._array("iterations"))
    converged = property(lambda self: self._array("converged"))
    final_delta = property(lambda self: self._array("final_delta"))
    failed_at = property(lambda self: self._array("failed_at"))
    admm_gap = property(lambda self: self._array("admm_gap"))
    elapsed = property(lambda self: self._array("elapsed"))

    @property
    def convergence_pct(self):
        return 100.0 * self.n_converged / self.n_pixels if self.n_pixels else 0.0


def _stats_from_batch(algorithm, b, y_dim, x_flat, wall):
    """RecoveryStats of a DeviceBatch: the aggregates by device reductions and
    one small copy; the per-pixel arrays stay on the device until read."""
    import torch
    it, fa, el = b.iterations, b.failed_at, b.elapsed
    cv = b.converged.bool()
    ok = fa < 0
    itl = it.to(torch.int64)
    agg = torch.stack([
        (cv & ok).sum().to(torch.float64),
        (~ok).sum().to(torch.float64),
        ((it == 0) & cv & ok).sum().to(torch.float64),
        torch.where(ok, itl, torch.zeros_like(itl)).sum().to(torch.float64),
        torch.where(ok, el, torch.zeros_like(el)).sum(),
    ]).cpu().tolist()
    n_failed = int(agg[1])
    failed = []
    if n_failed:
        idx = torch.nonzero(~ok).flatten()
        fav = fa[idx].cpu().numpy()
        failed = [(int(p // y_dim), int(p % y_dim), int(f)) for p, f in zip(idx.cpu().numpy(), fav)]
    st = RecoveryStats(
        n_pixels=int(it.numel()),
        n_converged=int(agg[0]),
        n_failed=n_failed,
        n_zero_pixels=int(agg[2]),
        total_iterations=int(agg[3]),
        recovery_time_s=float(agg[4]),
        failed_pixels=failed,
        algorithm=algorithm,
        wall_time_s=wall,
        _src={name: getattr(b, name) for name in _PER_PIXEL})
    st.results = _LazyResults(st, x_flat)
    return st


_STREAMS = {}


def _side_streams(device):
    """Per-device side streams of the host pipeline: H2D, two compute, D2H."""
    import torch
    key = str(device)
    if key not in _STREAMS:
        _STREAMS[key] = tuple(torch.cuda.Stream(device=device) for _ in range(4))
    return _STREAMS[key]


def _chunk_view(b, p0, p1):
    return DeviceBatch(x=b.x[p0:p1], iterations=b.iterations[p0:p1], converged=b.converged[p0:p1],
                       final_delta=b.final_delta[p0:p1], failed_at=b.failed_at[p0:p1],
                       admm_gap=b.admm_gap[p0:p1], lipschitz=b.lipschitz[p0:p1], elapsed=b.elapsed[p0:p1],
                       work=b.work[p0:p1])


def _raise_error_word(flag):
    """ValueErrors of the workspace error word (hcs_recover_status)."""
    if flag & 2:
        raise ValueError("mask entries must be strictly increasing band indices < N")
    if flag:
        raise ValueError("array must not contain infs or NaNs")


def _recover_host(algorithm, y_host, dictionary, config, x_host, chunk_pixels, stream):
    """Host buffers in and out, pipelined in pixel chunks: the H2D copy of
    chunk k+1 and the D2H copy of chunk k-1 run on their own streams while
    chunk k is solved; consecutive chunks alternate between two compute
    streams (each with its own workspace) so one launch's tail overlaps the
    next launch's start.  Results are identical to one launch (pixels are
    independent).  Returns the DeviceBatch of the whole cube (stats on the
    device) after every stream has finished."""
    import torch
    dev = torch.device("cuda", torch.cuda.current_device())
    P, m = int(y_host.shape[0]), int(y_host.shape[1])
    n = dictionary.n
    main = stream if stream is not None else torch.cuda.current_stream(dev)
    s_in, s_c0, s_c1, s_out = _side_streams(dev)
    lib = nat.load()
    algo = nat.ALGO_IDS[algorithm]
    f64 = dict(dtype=torch.float64, device=dev)
    with torch.cuda.stream(main):
        basis_d = torch.as_tensor(dictionary.basis, device=dev)
        y_d = torch.empty((P, m), **f64)
        masks_d = torch.empty((P, m), dtype=torch.uint8, device=dev)
        full = DeviceBatch(
            x=torch.empty((P, n), **f64), iterations=torch.empty((P,), dtype=torch.int32, device=dev),
            converged=torch.empty((P,), dtype=torch.uint8, device=dev), final_delta=torch.empty((P,), **f64),
            failed_at=torch.empty((P,), dtype=torch.int32, device=dev), admm_gap=torch.full((P,), math.nan, **f64),
            lipschitz=torch.full((P,), math.nan, **f64), elapsed=torch.empty((P,), **f64),
            work=torch.empty((P,), **f64))
        chunk = max(1, min(P, int(chunk_pixels)))
        # graded chunks: a short first chunk starts the solve after a short H2D,
        # a short last chunk leaves a short D2H after the last solve
        edge = min(chunk, max(1, P // 32))
        sizes = []
        if P >= 65536 and chunk > edge:
            mid = P - 2 * edge
            sizes = [edge] + [chunk] * (mid // chunk) + ([mid % chunk] if mid % chunk else []) + [edge]
        else:
            sizes = [chunk] * (P // chunk) + ([P % chunk] if P % chunk else [])
        bounds, p0 = [], 0
        for sz in sizes:
            bounds.append((p0, p0 + sz))
            p0 += sz
        wsb = lib.hcs_workspace_bytes(algo, chunk, n, m)
        ws = [torch.empty((max(wsb, 256),), dtype=torch.uint8, device=dev) for _ in range(min(2, len(bounds)))]
        errs = torch.zeros((max(1, len(bounds)),), dtype=torch.int32, device=dev)
        if dictionary.shared:
            masks_d.copy_(torch.as_tensor(dictionary.masks, device=dev).reshape(1, m).expand(P, m))
            mask_src = None
        else:
            if dictionary.masks.shape[0] != P:
                raise ValueError("per-pixel masks do not match the cube")
            mask_src = dictionary.pinned_masks()
    ready = torch.cuda.Event()
    ready.record(main)
    for s in (s_in, s_c0, s_c1, s_out):
        s.wait_event(ready)
    done_c = []

    def drain(k):
        p0, p1 = bounds[k]
        s_out.wait_event(done_c[k])
        with torch.cuda.stream(s_out):
            x_host[p0:p1].copy_(full.x[p0:p1], non_blocking=True)

    for k, (p0, p1) in enumerate(bounds):
        with torch.cuda.stream(s_in):
            y_d[p0:p1].copy_(y_host[p0:p1], non_blocking=True)
            if mask_src is not None:
                masks_d[p0:p1].copy_(mask_src[p0:p1], non_blocking=True)
            ev_in = torch.cuda.Event()
            ev_in.record(s_in)
        sc = s_c0 if k % 2 == 0 else s_c1
        sc.wait_event(ev_in)
        solve_batch(algorithm, y_d[p0:p1], masks_d[p0:p1], basis_d, config, stream=sc, workspace=ws[k % 2],
                    check_status=False, out=_chunk_view(full, p0, p1))
        with torch.cuda.stream(sc):
            errs[k].copy_(ws[k % 2][8:12].view(torch.int32)[0])
            ev = torch.cuda.Event()
            ev.record(sc)
        done_c.append(ev)
        if k >= 1:
            drain(k - 1)   # enqueued after chunk k so a blocking (pageable) copy overlaps its solve
    if bounds:
        drain(len(bounds) - 1)
    for s in (s_in, s_c0, s_c1, s_out):
        main.wait_stream(s)
    if bounds:   # the error word hcs_recover_status reads, per chunk
        _raise_error_word(int(((errs & 2).amax() | (errs & 1).amax()).item()))
    full.workspace = ws[0] if ws else None
    full.launches = sum(lib.hcs_recover_launches(algo, n, m, config.to_native()) for _ in bounds)
    return full


def recover_cube(measurements, dictionary, config, algorithm, jobs=1, stream=None, out=None, chunk_pixels=None):
    """Solve every pixel of an (x, y, m) measurement array (solvers.py:455-514).

    ``dictionary`` is a `Dictionary` with one shared mask (the reference's
    model) or per-pixel masks.  ``measurements`` may be a numpy array (the
    recovered cube comes back as float64 numpy), a host torch tensor (pinned
    for full copy speed; the cube comes back as a pinned host tensor) or a
    CUDA tensor (the cube stays on the device).  Host inputs are pipelined in
    chunks of ``chunk_pixels`` pixels (default: an eighth of the cube, at
    least 65,536) so host<->device copies overlap the solve.  ``out`` (host
    only): an (x, y, n) float64 C-contiguous numpy array or host tensor that
    receives the cube, avoiding a per-call allocation (pinning 3 GB costs
    ~1.6 s).  Failed pixels are flagged and left at zero."""
    import time
    import torch
    if algorithm not in SOLVERS:
        raise ValueError(f"unknown algorithm {algorithm!r}")
    is_torch = isinstance(measurements, torch.Tensor)
    on_device = is_torch and measurements.is_cuda
    if is_torch:
        if measurements.is_complex():
            raise ValueError("the GPU backend is real-valued")
        meas = measurements if measurements.dtype == torch.float64 else measurements.to(torch.float64)
    else:
        arr = np.asarray(measurements)
        if np.iscomplexobj(arr):
            if np.any(arr.imag != 0):
                raise ValueError("the GPU backend is real-valued")
            arr = arr.real
        meas = np.ascontiguousarray(arr, dtype=np.float64)
    if meas.ndim != 3:
        raise ValueError("measurements must be (x, y, m)")
    x_dim, y_dim, m = (int(s) for s in meas.shape)
    if not isinstance(dictionary, Dictionary):
        dictionary = Dictionary.from_matrix(dictionary.matrix)
    if m != dictionary.m:
        raise ValueError("measurement length does not match the dictionary")
    P = x_dim * y_dim
    n = dictionary.n
    if not dictionary.shared and dictionary.n_pixels != P:
        raise ValueError("per-pixel masks do not match the cube")
    if algorithm == "admm":
        dictionary.admm_factor(config.alpha)
    config.to_native()   # config errors before any device work
    if stream is not None:
        # everything below (solve, error flags, statistics reductions, the
        # copies) is ordered on the caller's stream
        with torch.cuda.stream(stream):
            return _recover_cube_on_stream(meas, is_torch, on_device, dictionary, config, algorithm, out,
                                           chunk_pixels, x_dim, y_dim, m, stream)
    return _recover_cube_on_stream(meas, is_torch, on_device, dictionary, config, algorithm, out, chunk_pixels,
                                   x_dim, y_dim, m, None)


def _recover_cube_on_stream(meas, is_torch, on_device, dictionary, config, algorithm, out, chunk_pixels, x_dim,
                            y_dim, m, stream):
    import time
    import torch
    P = x_dim * y_dim
    n = dictionary.n
    t0 = time.perf_counter()
    if on_device:
        if out is not None:
            raise ValueError("out= is for host measurements")
        y_d = meas.reshape(P, m).contiguous()
        basis_d, masks_d = dictionary.device_arrays(y_d.device, P)
        b = solve_batch(algorithm, y_d, masks_d, basis_d, config, stream=stream)
        cube = b.x.reshape(x_dim, y_dim, n)
    else:
        y_host = meas.reshape(P, m).contiguous() if is_torch else torch.from_numpy(meas.reshape(P, m))
        if out is not None:
            ret = out
            x_host = torch.from_numpy(out) if isinstance(out, np.ndarray) else out
            if (tuple(x_host.shape) != (x_dim, y_dim, n) or x_host.dtype != torch.float64
                    or x_host.is_cuda or not x_host.is_contiguous()):
                raise ValueError(f"out must be a C-contiguous float64 host array of shape {(x_dim, y_dim, n)}")
        elif is_torch:
            x_host = ret = torch.empty((x_dim, y_dim, n), dtype=torch.float64, pin_memory=True)
        else:
            ret = np.empty((x_dim, y_dim, n), dtype=np.float64)
            x_host = torch.from_numpy(ret)
        if chunk_pixels is None:
            chunk_pixels = max(65536, -(-P // 8))
        b = _recover_host(algorithm, y_host, dictionary, config, x_host.reshape(P, n), chunk_pixels, stream)
        cube = ret
    wall = time.perf_counter() - t0
    x_flat = cube.reshape(P, n)
    return cube, _stats_from_batch(algorithm, b, y_dim, x_flat, wall)
