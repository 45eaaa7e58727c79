"""Parity comparator of SURVEY.md §8(c), shared by the CPU and GPU tests.

Criteria per pixel, candidate vs reference:
  1. coefficients: ||x_c - x_r|| <= RTOL * ||x_r||  (||x_c|| <= 1e-12 if x_r = 0);
  2. significant support {i : |x_i| > 1e-10 ||x||} identical;
  3. iterations / converged / failed_at identical;
unless the pixel is a *tie exception*: the first argmax_k call at which the two
selection traces differ is roundoff-degenerate on the reference side
(max|v| <= TIE * ||y||, or k-th gap <= TIE * ||y||).  Tie exceptions are
counted and reported, never silently dropped.  When the candidate's trace is
unknown, `forced replay` (tests that have it) closes the hole described in
SURVEY.md §8(c).
"""

import math

import numpy as np

RTOL = 1e-9          # north_star: coefficients within 1e-9 relative (FP64)
SUPPORT_REL = 1e-10
TIE = 1e-12


def significant(x):
    nrm = np.linalg.norm(x)
    if nrm == 0.0:
        return np.zeros(x.shape, dtype=bool)
    return np.abs(x) > SUPPORT_REL * nrm


def coef_ok(xc, xr):
    nr = np.linalg.norm(xr)
    if nr == 0.0:
        return np.linalg.norm(xc) <= 1e-12
    return np.linalg.norm(xc - xr) <= RTOL * nr


def first_divergence(trace_r, trace_c):
    """Index of the first argmax_k call whose selection differs, or None."""
    for i, (a, b) in enumerate(zip(trace_r, trace_c)):
        if int(a[0]) != int(b[0]) or tuple(a[1]) != tuple(b[1]):
            return i
    if len(trace_r) != len(trace_c):
        return min(len(trace_r), len(trace_c))
    return None


def degenerate(entry, ynorm):
    """Roundoff-degenerate selection on the reference side."""
    _, _, vmax, gap = entry
    return vmax <= TIE * ynorm or gap <= TIE * ynorm


def replay_matches(res, cand, p):
    """Forced-selection replay result vs the candidate pixel p."""
    return (int(res.iterations) == int(cand["iterations"][p]) and bool(res.converged) == bool(cand["converged"][p])
            and int(res.failed_at) == int(cand["failed_at"][p]) and coef_ok(cand["x"][p], res.x)
            and np.array_equal(significant(cand["x"][p]), significant(res.x)))


def compare(ref, cand, y, ref_traces=None, cand_traces=None, algo="", replay=None):
    """ref/cand: dicts with x, iterations, converged, failed_at arrays.

    ``replay(p, force)`` (optional) re-runs the oracle on pixel p with the
    candidate's selections forced at roundoff-degenerate calls; a tie
    exception is only accepted if that replay reproduces the candidate.
    Returns a report dict; ``report["bad"]`` lists real mismatches."""
    P = len(ref["iterations"])
    bad, ties, worst = [], [], 0.0
    for p in range(P):
        xr, xc = ref["x"][p], cand["x"][p]
        ok_fail = int(ref["failed_at"][p]) == int(cand["failed_at"][p])
        same_it = (int(ref["iterations"][p]) == int(cand["iterations"][p])
                   and bool(ref["converged"][p]) == bool(cand["converged"][p]))
        nr = np.linalg.norm(xr)
        rel = np.linalg.norm(xc - xr) / nr if nr > 0 else np.linalg.norm(xc)
        good = ok_fail and same_it and coef_ok(xc, xr) and np.array_equal(significant(xc), significant(xr))
        if good:
            worst = max(worst, rel)
            continue
        why = dict(pixel=p, rel=float(rel), it_ref=int(ref["iterations"][p]),
                   it_cand=int(cand["iterations"][p]))
        if ref_traces is not None and ok_fail:
            ynorm = float(np.linalg.norm(np.nan_to_num(y[p])))
            tr = ref_traces[p]
            if cand_traces is not None:
                i = first_divergence(tr, cand_traces[p])
                if i is not None and i < len(tr) and degenerate(tr[i], ynorm):
                    entry = dict(why, call=i, vmax=tr[i][2] / ynorm, gap=tr[i][3] / ynorm)
                    if replay is not None:
                        force = {c: tuple(e[1]) for c, e in enumerate(cand_traces[p])}
                        entry["replay_ok"] = replay_matches(replay(p, force), cand, p)
                        if not entry["replay_ok"]:
                            bad.append(dict(entry, reason="forced-selection replay does not reproduce"))
                            continue
                    ties.append(entry)
                    continue
            elif any(degenerate(e, ynorm) for e in tr):
                ties.append(dict(why, call=-1))
                continue
        bad.append(why)
    return dict(algo=algo, pixels=P, bad=bad, ties=ties, worst_rel=worst)


def load_traces(blob):
    import json
    return json.loads(str(blob))


def psnr_close(p_ref, p_cand, mse_ref, mse_cand, peak):
    """|dPSNR| <= 0.01 dB outside the roundoff regime (PSNR_ref < 200 dB);
    inside it both MSEs must be <= 1e-25 * peak^2."""
    if p_ref < 200.0:
        return abs(p_ref - p_cand) <= 0.01
    return mse_ref <= 1e-25 * peak * peak and mse_cand <= 1e-25 * peak * peak


def psnr(ref, rec):
    peak = float(np.abs(ref).max())
    mse = float(np.mean((ref - rec) ** 2))
    return (math.inf if mse == 0 else 10 * math.log10(peak * peak / mse)), mse, peak
