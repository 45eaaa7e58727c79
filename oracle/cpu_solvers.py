"""CPU ORACLE -- TEST INFRASTRUCTURE ONLY.

Real-FP64 numpy/scipy restatement of the reference's per-pixel recovery
(`/root/reference/pkg/src/hypercs/{kernels,solvers,transform}.py`).  Only
`tests/`, `__graft_entry__.smoke()` and `bench.py`'s CPU-baseline leg may
import this module, and only as the checker / the timed CPU baseline: the
product path (`paper_2401_14762_b200`) never imports it and has no CPU
fallback.

What is restated, and where it comes from:

* soft threshold            kernels.py:14-28   v * (max(|v|-t, 0) / |v|), 0 at v = 0
* top-k selection           kernels.py:31-41   stable argsort of -|v|, first k, sorted
* least squares             kernels.py:44-67   pivoted QR + triangular solve; gelsd
                                              minimum-norm fallback below RANK_RTOL
* residual delta            kernels.py:70-76
* power-iteration Lipschitz transform.py:176-217
* ADMM factor               transform.py:253-264 (Cholesky of A^T A + alpha I)
* stop rule                 solvers.py:115-127 (delta < eps > timeout > cap, delta0 = 1)
* fista / admm / gomp / biht / cosamp  solvers.py:164-394
* y = 0 shortcut, non-finite failure   solvers.py:145-157
* sparsify (mean/std rule)  transform.py:73-97 (keep (|x| - mean) >= factor * std)
* input side of a cube      cli.py:97-139 with the DCT basis, per-pixel masks and the
                            BASELINE T max|c| rule (the synth.py v1 recipe)

Deviations (all documented in DESIGN.md): real FP64 instead of complex128
(the imaginary parts are identically zero for real bases);
the wall-clock budget is not modelled (time_limit=None, `max_iter` caps only);
per-pixel dictionaries A_p = Psi[mask_p, :] instead of one shared dictionary.

Parity pin: `tests/golden/*.npz` hold outputs of the reference package itself
(`tests/golden/make_golden.py` imports /root/reference in the build container);
`tests/test_oracle_golden.py` checks this restatement against them.

Every argmax_k call can be recorded in a ``trace`` list for the tie
classification of SURVEY.md §8(c): entries are
(k, selected indices, max|v|, gap between the k-th and (k+1)-th magnitude).
"""

import math
import os
import time
from concurrent.futures import ProcessPoolExecutor
from dataclasses import dataclass

import numpy as np
import scipy.linalg

RANK_RTOL = 1e-10          # kernels.py:11
POWER_ITER_CAP = 1000      # transform.py:15
POWER_ITER_RTOL = 1e-10    # transform.py:16

ALGORITHMS = ("fista", "admm", "gomp", "biht", "cosamp")


@dataclass(frozen=True)
class OracleConfig:
    """Solver parameters (solvers.py:40-85), time_limit fixed to None."""

    lam: float = 0.1
    kappa: int = 1
    atoms_per_iter: int = 0      # 0 -> max(1, kappa // 5)  (solvers.py:72-73)
    mu: float = 0.1
    alpha: float = 1.8
    epsilon: float = 1e-8
    max_iter: int = 0            # 0 -> no cap

    @property
    def G(self):
        return self.atoms_per_iter if self.atoms_per_iter > 0 else max(1, self.kappa // 5)


# --------------------------------------------------------------------------- kernels


def soft_threshold(v, t):
    """kernels.py:14-28."""
    if t < 0:
        raise ValueError("threshold must be >= 0")
    v = np.asarray(v, dtype=np.float64)
    mag = np.abs(v)
    scale = np.zeros_like(mag)
    pos = mag > 0
    scale[pos] = np.maximum(mag[pos] - t, 0.0) / mag[pos]
    return v * scale


TIE_REL = 1e-12   # roundoff-degenerate selection: max|v| or k-th gap <= TIE_REL * ||y||


class Recorder(list):
    """Selection trace; with ``force`` it also implements the forced-selection
    replay of SURVEY.md §8(c): at a call whose own selection is
    roundoff-degenerate (max|v| or the k-th gap <= TIE_REL * ||y||) the
    selection recorded by the candidate implementation (force[call index]) is
    used instead of the oracle's own."""

    def __init__(self, force=None, ynorm=0.0):
        super().__init__()
        self.force = force or {}
        self.ynorm = ynorm
        self.forced = 0


def argmax_k(v, k, trace=None):
    """kernels.py:31-41: k largest |v|, ties to the lowest index, ascending."""
    v = np.asarray(v)
    if k < 1 or k > v.size:
        raise ValueError(f"k must be in [1, {v.size}], got {k}")
    mag = np.abs(v)
    order = np.argsort(-mag, kind="stable")
    picked = np.sort(order[:k])
    if trace is not None:
        srt = mag[order]
        gap = float(srt[k - 1] - srt[k]) if k < v.size else math.inf
        vmax = float(srt[0])
        if isinstance(trace, Recorder) and len(trace) in trace.force:
            lim = TIE_REL * trace.ynorm
            forced = tuple(int(i) for i in trace.force[len(trace)])
            if (vmax <= lim or gap <= lim) and len(forced) == k:
                picked = np.array(forced, dtype=np.intp)
                trace.forced += 1
        trace.append((k, tuple(int(i) for i in picked), vmax, gap))
    return picked


def least_squares(b, y):
    """kernels.py:44-67: column-pivoted QR solve, min-norm gelsd fallback."""
    b = np.asarray(b, dtype=np.float64)
    y = np.asarray(y, dtype=np.float64)
    if b.ndim != 2:
        raise ValueError("matrix must be 2-D")
    if y.shape != (b.shape[0],):
        raise ValueError("right-hand side length does not match the matrix")
    m, k = b.shape
    q, r, piv = scipy.linalg.qr(b, mode="economic", pivoting=True)
    d = np.abs(np.diag(r))
    if m >= k and d.size == k and d.min() > RANK_RTOL * d.max():
        z = scipy.linalg.solve_triangular(r, q.T @ y)
        s = np.empty_like(z)
        s[piv] = z
        return s
    s = scipy.linalg.lstsq(b, y, cond=RANK_RTOL, lapack_driver="gelsd")[0]
    return s


def residual_delta(r, r_prev):
    """kernels.py:70-76."""
    return float(np.linalg.norm(np.asarray(r) - np.asarray(r_prev)))


def lipschitz(a, max_iter=POWER_ITER_CAP, rtol=POWER_ITER_RTOL):
    """transform.py:176-217: largest eigenvalue of A^T A by power iteration
    from the normalised all-ones vector, with the A^T 1 restart."""
    a = np.asarray(a, dtype=np.float64)
    m, n = a.shape

    def gram(v):
        return a.T @ (a @ v)

    v = np.full(n, 1.0 / np.sqrt(n))
    w = gram(v)
    nw = np.linalg.norm(w)
    if nw < 1e-300:
        v = a.T @ np.ones(m)
        nv = np.linalg.norm(v)
        if nv < 1e-300:
            rng = np.random.default_rng(0)
            v = rng.standard_normal(n)
            nv = np.linalg.norm(v)
        v = v / nv
        w = gram(v)
        nw = np.linalg.norm(w)
        if nw < 1e-300:
            return 0.0
    est = float(v @ w)
    for _ in range(max_iter):
        v = w / nw
        w = gram(v)
        nw = np.linalg.norm(w)
        if nw < 1e-300:
            return 0.0
        new = float(v @ w)
        if abs(new - est) <= rtol * abs(new):
            return new
        est = new
    return est


# --------------------------------------------------------------------------- solvers


@dataclass
class PixelResult:
    x: np.ndarray
    iterations: int
    converged: bool
    final_delta: float
    admm_gap: float = math.nan
    failed_at: int = -1          # iteration of a NumericalFailure, -1 if none
    lipschitz: float = math.nan
    elapsed: float = 0.0         # seconds spent on the pixel (dictionary + solve)


class _Failure(Exception):
    def __init__(self, iteration):
        super().__init__(iteration)
        self.iteration = iteration


def _iterate(step, y, cfg):
    """Shared loop of solvers.py: stop rule before every pass (solvers.py:115-127);
    ``step(residual)`` returns (new residual, or None for the support>m break).
    Returns (iterations, converged, delta)."""
    residual = y
    delta = 1.0
    iterations = 0
    while True:
        if delta < cfg.epsilon:
            return iterations, True, delta
        if cfg.max_iter and iterations >= cfg.max_iter:
            return iterations, False, delta
        new = step(residual)
        if new is None:                      # support outgrew m: keep the last iterate
            return iterations, False, delta
        delta = residual_delta(new, residual)
        residual = new
        iterations += 1
        if not (math.isfinite(delta) and step.finite()):
            raise _Failure(iterations)


class _Step:
    """Callable solver pass holding the iterate; finite() checks the iterate
    the reference passes to _check_finite."""

    def finite(self):
        return bool(np.isfinite(self.checked()).all())


class _Fista(_Step):
    # solvers.py:164-203
    def __init__(self, a, y, cfg, lip):
        self.a, self.y = a, y
        self.inv_l = 1.0 / lip
        self.thr = cfg.lam * self.inv_l
        n = a.shape[1]
        self.x = np.zeros(n)
        self.z = self.x
        self.t = 1.0

    def __call__(self, residual):
        a = self.a
        grad = a.T @ (a @ self.z - self.y)
        x_new = soft_threshold(self.z - self.inv_l * grad, self.thr)
        t_new = 0.5 * (1.0 + math.sqrt(1.0 + 4.0 * self.t * self.t))
        self.z = x_new + ((self.t - 1.0) / t_new) * (x_new - self.x)
        self.x, self.t = x_new, t_new
        return self.y - a @ self.x

    def checked(self):
        return self.x


class _Admm(_Step):
    # solvers.py:206-245, factor from transform.py:253-264
    def __init__(self, a, y, cfg):
        self.a, self.y, self.alpha = a, y, cfg.alpha
        n = a.shape[1]
        gram = a.T @ a
        gram[np.diag_indices_from(gram)] += cfg.alpha
        self.factor = scipy.linalg.cho_factor(gram)
        self.aty = a.T @ y
        self.thr = cfg.lam / cfg.alpha
        self.x = np.zeros(n)
        self.z = np.zeros(n)
        self.w = np.zeros(n)

    def __call__(self, residual):
        self.x = scipy.linalg.cho_solve(self.factor, self.aty + self.alpha * (self.z - self.w))
        self.z = soft_threshold(self.x + self.w, self.thr)
        self.w = self.w + self.x - self.z
        return self.y - self.a @ self.x

    def checked(self):
        return self.z


class _Gomp(_Step):
    # solvers.py:248-297
    def __init__(self, a, y, cfg, trace):
        self.a, self.y, self.cfg, self.trace = a, y, cfg, trace
        self.support = np.empty(0, dtype=np.intp)
        self.x = np.zeros(a.shape[1])

    def __call__(self, residual):
        a, y = self.a, self.y
        m, n = a.shape
        picks = argmax_k(a.T @ residual, self.cfg.G, self.trace)
        self.support = np.union1d(self.support, picks)
        if self.support.size > m:
            return None
        full = np.zeros(n)
        full[self.support] = least_squares(a[:, self.support], y)
        top = argmax_k(full, self.cfg.kappa, self.trace)
        self.x = np.zeros(n)
        self.x[top] = least_squares(a[:, top], y)
        return y - a @ self.x

    def checked(self):
        return self.x


class _Biht(_Step):
    # solvers.py:300-342
    def __init__(self, a, y, cfg, trace):
        self.a, self.y, self.cfg, self.trace = a, y, cfg, trace
        self.x = np.zeros(a.shape[1])

    def __call__(self, residual):
        a, y, kappa = self.a, self.y, self.cfg.kappa
        m, n = a.shape
        u = self.x + self.cfg.mu * (a.T @ (y - a @ self.x))
        cand = np.union1d(argmax_k(u, kappa, self.trace), np.flatnonzero(self.x))
        if cand.size > m:
            return None
        s = least_squares(a[:, cand], y)
        keep = argmax_k(s, min(kappa, s.size), self.trace)
        pruned = np.zeros_like(s)
        pruned[keep] = s[keep]
        self.x = np.zeros(n)
        self.x[cand] = pruned
        return y - a @ self.x

    def checked(self):
        return self.x


class _Cosamp(_Step):
    # solvers.py:345-394
    def __init__(self, a, y, cfg, trace):
        self.a, self.y, self.cfg, self.trace = a, y, cfg, trace
        self.support = np.empty(0, dtype=np.intp)
        self.x = np.zeros(a.shape[1])

    def __call__(self, residual):
        a, y, kappa = self.a, self.y, self.cfg.kappa
        m, n = a.shape
        self.support = np.union1d(self.support, argmax_k(a.T @ residual, 2 * kappa, self.trace))
        if self.support.size > m:
            return None
        s = least_squares(a[:, self.support], y)
        keep = argmax_k(s, min(kappa, s.size), self.trace)
        self.support = self.support[keep]
        self.x = np.zeros(n)
        self.x[self.support] = s[keep]
        return y - a @ self.x

    def checked(self):
        return self.x


def check_preconditions(algo, m, n, cfg):
    """Per-solver ValueErrors (solvers.py:259-260, 306-307, 355-358)."""
    if algo == "gomp" and not cfg.G <= cfg.kappa <= m:
        raise ValueError(f"need atoms_per_iter <= kappa <= {m}")
    if algo == "biht" and cfg.kappa > m:
        raise ValueError(f"kappa must be <= {m}")
    if algo == "cosamp":
        if 2 * cfg.kappa > n:
            raise ValueError(f"need 2 * kappa <= {n}")
        if cfg.kappa > m:
            raise ValueError(f"kappa must be <= {m}")


def solve_pixel(algo, y, a, cfg, trace=None, lip=None):
    """One pixel: SOLVERS[algo](y, Dictionary.from_matrix(a), cfg) in real FP64."""
    a = np.asarray(a, dtype=np.float64)
    y = np.asarray(y, dtype=np.float64)
    m, n = a.shape
    if y.shape != (m,):
        raise ValueError("measurement length does not match the dictionary")
    check_preconditions(algo, m, n, cfg)
    if lip is None:
        lip = lipschitz(a)
    if not y.any():
        # _zero_result carries no admm_gap (solvers.py:145-152)
        return PixelResult(np.zeros(n), 0, True, 0.0, math.nan, lipschitz=lip)
    if algo == "fista":
        step = _Fista(a, y, cfg, lip)
    elif algo == "admm":
        step = _Admm(a, y, cfg)
    elif algo == "gomp":
        step = _Gomp(a, y, cfg, trace)
    elif algo == "biht":
        step = _Biht(a, y, cfg, trace)
    elif algo == "cosamp":
        step = _Cosamp(a, y, cfg, trace)
    else:
        raise ValueError(f"unknown algorithm {algo!r}")
    try:
        its, conv, delta = _iterate(step, y, cfg)
    except _Failure as f:
        return PixelResult(np.zeros(n), 0, False, math.nan, failed_at=f.iteration, lipschitz=lip)
    gap = float(np.linalg.norm(step.x - step.z)) if algo == "admm" else math.nan
    out = step.z.copy() if algo == "admm" else step.x.copy()
    return PixelResult(out, its, conv, delta, gap, lipschitz=lip)


# --------------------------------------------------------------------------- cubes


@dataclass
class CubeResult:
    x: np.ndarray            # (P, n)
    iterations: np.ndarray   # (P,) int32
    converged: np.ndarray    # (P,) bool
    final_delta: np.ndarray  # (P,)
    admm_gap: np.ndarray     # (P,)
    failed_at: np.ndarray    # (P,) int32, -1 ok
    lipschitz: np.ndarray    # (P,)
    traces: list | None = None
    elapsed: np.ndarray | None = None   # (P,) seconds per pixel


def single_thread_blas():
    """Pool initializer: one BLAS thread per worker process."""
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    try:
        from threadpoolctl import threadpool_limits
        threadpool_limits(1)
    except ImportError:
        pass


def _solve_range(args):
    algo, basis, y, masks, cfg, want_trace = args
    out = []
    for p in range(y.shape[0]):
        trace = [] if want_trace else None
        t0 = time.perf_counter()
        a = basis[masks[p].astype(np.intp), :]
        r = solve_pixel(algo, y[p], a, cfg, trace)
        r.elapsed = time.perf_counter() - t0     # SolverResult.elapsed semantics (solvers.py:166, 201)
        out.append((r, trace))
    return out


def solve_cube(algo, basis, y, masks, cfg, jobs=1, trace=False, chunk=64, pool=None):
    """Per-pixel oracle over a (P, m) measurement array with per-pixel masks:
    the reference's SOLVERS[algo] on Dictionary.from_matrix(Psi[mask_p]).
    ``pool``: an existing process pool to reuse (else one is made for jobs > 1)."""
    y = np.asarray(y, dtype=np.float64)
    masks = np.asarray(masks)
    P, m = y.shape
    n = basis.shape[0]
    check_preconditions(algo, m, n, cfg)
    items = [(algo, basis, y[i:i + chunk], masks[i:i + chunk], cfg, trace)
             for i in range(0, P, chunk)]
    if pool is not None:
        parts = list(pool.map(_solve_range, items))
    elif jobs == 1 or P <= chunk:
        parts = [_solve_range(it) for it in items]
    else:
        with ProcessPoolExecutor(max_workers=jobs, initializer=single_thread_blas) as pool:
            parts = list(pool.map(_solve_range, items))
    flat = [r for part in parts for r in part]
    return CubeResult(
        x=np.stack([r.x for r, _ in flat]) if flat else np.zeros((0, n)),
        iterations=np.array([r.iterations for r, _ in flat], dtype=np.int32),
        converged=np.array([r.converged for r, _ in flat], dtype=bool),
        final_delta=np.array([r.final_delta for r, _ in flat]),
        admm_gap=np.array([r.admm_gap for r, _ in flat]),
        failed_at=np.array([r.failed_at for r, _ in flat], dtype=np.int32),
        lipschitz=np.array([r.lipschitz for r, _ in flat]),
        traces=[t for _, t in flat] if trace else None,
        elapsed=np.array([r.elapsed for r, _ in flat]),
    )


def psnr(reference, reconstruction):
    """metrics.py:30-55 with the default abs-max peak; inf when identical."""
    ref = np.asarray(reference, dtype=np.float64)
    rec = np.asarray(reconstruction, dtype=np.float64)
    peak = float(np.abs(ref).max())
    if peak <= 0:
        raise ValueError("non-positive peak")
    mse = float(np.mean((ref - rec) ** 2))
    return math.inf if mse == 0.0 else 10.0 * math.log10(peak * peak / mse)


# ---------------------------------------------------------------- input side


def sparsify(x, factor):
    """transform.py:73-97: zero x_i where (|x_i| - mean|x|) < factor * std|x|
    (population std); kept entries bit-identical.  Returns (out, mean, std,
    zero_fraction)."""
    if factor < 0:
        raise ValueError("threshold factor must be >= 0")
    x = np.asarray(x, dtype=np.float64)
    if x.size == 0:
        raise ValueError("cannot sparsify an empty vector")
    mags = np.abs(x)
    mean = float(mags.mean())
    std = float(mags.std())
    keep = (mags - mean) >= factor * std
    return np.where(keep, x, 0.0), mean, std, 1.0 - float(keep.mean())


def sparsify_measure(spectra, basis, masks, rule="maxrel", factor=0.1):
    """Input side of a cube for the DCT basis (cli.py:97-139 restated):
    c = basis^T f, threshold (maxrel: |c| < factor max|c| -> 0; meanstd: the
    sparsify rule), f_s = basis c, y = f_s[mask].  Returns (coeffs, f_s, y)."""
    c = np.asarray(spectra, dtype=np.float64) @ basis
    mag = np.abs(c)
    if rule == "maxrel":
        c[mag < factor * mag.max(axis=1, keepdims=True)] = 0.0
    else:
        mean = mag.mean(axis=1, keepdims=True)
        std = mag.std(axis=1, keepdims=True)
        c[(mag - mean) < factor * std] = 0.0
    fs = c @ basis.T
    return c, fs, np.take_along_axis(fs, np.asarray(masks, dtype=np.intp), axis=1)
