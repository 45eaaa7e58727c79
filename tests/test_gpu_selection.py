"""GPU: the CTA top-k selection used by the greedy solvers (radix select) against
argmax_k of the reference (kernels.py:31-41, restated by the oracle) and the
ranking implementation it replaced -- exact set equality, including exact
ties, zeros, signed zeros, NaN and infinities."""

import ctypes

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import cpu_solvers as oc  # noqa: E402
from paper_2401_14762_b200 import _native  # noqa: E402

pytestmark = pytest.mark.gpu


def gpu_topk(v, k, variant):
    lib = _native.load()
    batch, n = v.shape
    dv = torch.as_tensor(np.ascontiguousarray(v), device="cuda")
    bm = torch.zeros((batch, 8), dtype=torch.int32, device="cuda")
    rc = lib.hcs_debug_cta_topk(ctypes.c_void_p(dv.data_ptr()), batch, n, k, ctypes.c_void_p(bm.data_ptr()), variant)
    assert rc == 0
    bits = np.unpackbits(bm.cpu().numpy().view(np.uint8), axis=1, bitorder="little")
    return [tuple(np.flatnonzero(b)) for b in bits]


def vectors(n, seed):
    rng = np.random.default_rng(seed)
    out = [rng.standard_normal(n)]
    t = np.round(rng.standard_normal(n), 1)             # many exact ties
    out.append(t)
    z = rng.standard_normal(n)
    z[rng.random(n) < 0.5] = 0.0                       # zeros, some negative zeros
    z[rng.random(n) < 0.2] = -0.0
    out.append(z)
    s = rng.standard_normal(n)
    s[rng.random(n) < 0.1] = np.nan
    s[rng.random(n) < 0.05] = np.inf
    s[rng.random(n) < 0.05] = -np.inf
    out.append(s)
    c = np.full(n, 3.0)                                # all equal
    c[::3] *= -1
    out.append(c)
    e = rng.standard_normal(n) * 1e-300                # tiny / subnormal magnitudes
    e[::4] = 5e-324
    out.append(e)
    return np.stack(out)


@pytest.mark.parametrize("n", [1, 7, 33, 66, 81, 224, 256])
def test_cta_topk_matches_argmax_k(n):
    v = vectors(n, n)
    for k in sorted(k for k in {1, 2, 5, n // 3, n // 2, n - 1, n} if 1 <= k <= n):
        got = gpu_topk(v, k, 1)
        old = gpu_topk(v, k, 0)
        for row in range(v.shape[0]):
            want = tuple(int(i) for i in oc.argmax_k(v[row], k))
            assert got[row] == want, (n, k, row)
            assert old[row] == want, (n, k, row)


@pytest.mark.parametrize("mode", [0, 1, 2])
def test_fast_division_is_ddiv_rn(mode):
    """The branch-free division of the convex epilogues (ddiv_fast / soft_fast,
    hcs_common.cuh) against __ddiv_rn / soft on 2^28 operand pairs: every
    quotient it accepts is bit-identical; pairs outside its range are rejected
    (redone with __ddiv_rn by the caller).  Modes: moderate exponents, the full
    bit range (subnormals, infinities, NaN), soft-threshold operands."""
    lib = _native.load()
    lib.hcs_debug_divcheck.argtypes = [ctypes.c_ulonglong, ctypes.c_ulonglong, ctypes.c_int,
                                       ctypes.POINTER(ctypes.c_ulonglong)]
    out = (ctypes.c_ulonglong * 3)()
    assert lib.hcs_debug_divcheck(1 << 28, 777 + mode, mode, out) == 0
    accepted, different, rejected = out[0], out[1], out[2]
    assert accepted + rejected == 1 << 28
    assert different == 0
    if mode != 1:
        assert rejected == 0          # ordinary operands always take the fast path
    else:
        assert accepted > (1 << 27)   # and most of the full bit range too
