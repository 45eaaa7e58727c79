"""C-ABI hardening and the round-1 advisor findings, on the GPU.

* masks are validated on the device: an entry >= N or a non-increasing row
  makes hcs_recover_status return HCS_EINVAL (ValueError in Python) and no
  solver kernel reads the masks (transform.py:106-113 semantics);
* hcs_check_basis measures max |Psi^T Psi - I| (orthonormality is a
  precondition of the closed forms; the header documents the violation as
  undefined behaviour);
* FISTA / ADMM at sampling ratios whose 32-slot layout exceeds one SM's
  shared memory (N = 224, M = 134 and 224) fall back to the 16-slot engine;
* batched least squares beyond shared memory (128 x 128, 224 x 100) run from
  a global scratch and match numpy;
* recover_cube(stream=s) orders the solve, the error word and the statistics
  on s;
* parallel.recover_cube_sharded without a process group equals recover_cube.
"""

import ctypes

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import paper_2401_14762_b200 as hcs  # noqa: E402
from oracle import cpu_solvers as oc  # noqa: E402
from paper_2401_14762_b200 import _native as nat  # noqa: E402
from paper_2401_14762_b200 import kernels as gk  # noqa: E402
from paper_2401_14762_b200 import parallel, synth  # noqa: E402
from paper_2401_14762_b200.solvers import SolverConfig, recover_cube, solve_batch  # noqa: E402
from paper_2401_14762_b200.transform import Dictionary  # noqa: E402

pytestmark = pytest.mark.gpu


def _cube(P=64, n=224, seed=3):
    return synth.generate(P // 8, 8, n, seed=seed)


def _raw_recover(algo, y, masks, basis, prm):
    """hcs_recover straight through ctypes (a C caller's view)."""
    lib = nat.load()
    P, m = y.shape
    n = basis.shape[0]
    dev = torch.device("cuda")
    yd, md, bd = (torch.as_tensor(a, device=dev) for a in (y, masks, basis))
    x = torch.empty((P, n), dtype=torch.float64, device=dev)
    it = torch.empty(P, dtype=torch.int32, device=dev)
    cv = torch.empty(P, dtype=torch.uint8, device=dev)
    fd = torch.empty(P, dtype=torch.float64, device=dev)
    fa = torch.empty(P, dtype=torch.int32, device=dev)
    st = nat.HcsStats(iterations=it.data_ptr(), converged=cv.data_ptr(), final_delta=fd.data_ptr(),
                      failed_at=fa.data_ptr())
    wsb = lib.hcs_workspace_bytes(algo, P, n, m)
    ws = torch.empty(max(wsb, 256), dtype=torch.uint8, device=dev)
    code = lib.hcs_recover(algo, P, n, m, bd.data_ptr(), yd.data_ptr(), md.data_ptr(), prm,
                           x.data_ptr(), st, ws.data_ptr(), ws.numel(), None)
    assert code == nat.HCS_OK, lib.hcs_last_error()
    return lib.hcs_recover_status(ws.data_ptr(), None), lib.hcs_last_error()


@pytest.mark.parametrize("algo", [0, 1, 2, 3, 4])
@pytest.mark.parametrize("defect", ["out_of_range", "not_increasing"])
def test_bad_masks_are_rejected_through_the_abi(algo, defect):
    c = _cube(n=154)
    masks = c.masks.copy()
    if defect == "out_of_range":
        masks[5, -1] = 200          # >= N = 154: a read past the basis if it were used
    else:
        masks[7, 3] = masks[7, 2]   # repeated band
    prm = nat.HcsParams(lam=0.1, mu=0.1, alpha=1.8, epsilon=1e-8, kappa=12, atoms_per_iter=0, max_iter=50)
    code, msg = _raw_recover(algo, c.y, masks, c.basis, prm)
    assert code == nat.HCS_EINVAL and b"mask" in msg
    # the same call with valid masks is fine
    code, _ = _raw_recover(algo, c.y, c.masks, c.basis, prm)
    assert code == nat.HCS_OK


def test_bad_masks_raise_valueerror_in_python():
    c = _cube(n=154)
    masks = c.masks.copy()
    masks[0, 0], masks[0, 1] = masks[0, 1], masks[0, 0]
    dev = torch.device("cuda")
    with pytest.raises(ValueError, match="mask"):
        solve_batch("gomp", torch.as_tensor(c.y, device=dev), torch.as_tensor(masks, device=dev),
                    torch.as_tensor(c.basis, device=dev), SolverConfig(kappa=12, time_limit=None))


def test_check_basis_measures_orthonormality():
    lib = nat.load()
    b = synth.dct_basis(224)
    out = ctypes.c_double()
    assert lib.hcs_check_basis(224, torch.as_tensor(b, device="cuda").data_ptr(), ctypes.byref(out), None) == 0
    assert out.value < 1e-13
    bad = b.copy()
    bad[3, 5] += 1e-3
    assert lib.hcs_check_basis(224, torch.as_tensor(bad, device="cuda").data_ptr(), ctypes.byref(out), None) == 0
    assert 1e-4 < out.value < 1e-2


@pytest.mark.parametrize("ratio", [0.6, 1.0])
@pytest.mark.parametrize("algo,params", [("fista", dict(lam=0.1)), ("admm", dict(lam=0.1, alpha=1.8))])
def test_high_sampling_ratios_use_the_16_slot_engine(ratio, algo, params):
    n, P = 224, 80
    rng = np.random.default_rng(5)
    m = int(np.floor(ratio * n + 0.5))
    c = synth.generate(10, 8, n, seed=9)
    masks = np.sort(np.argsort(rng.random((P, n)), axis=1)[:, :m], axis=1).astype(np.uint8)
    y = np.take_along_axis(c.spectra, masks.astype(np.intp), axis=1)
    dev = torch.device("cuda")
    cfg = SolverConfig(time_limit=None, max_iter=3000, **params)
    b = solve_batch(algo, torch.as_tensor(y, device=dev), torch.as_tensor(masks, device=dev),
                    torch.as_tensor(c.basis, device=dev), cfg)
    ref = oc.solve_cube(algo, c.basis, y, masks, oc.OracleConfig(max_iter=3000, **params), jobs=8)
    np.testing.assert_array_equal(b.iterations.cpu().numpy(), ref.iterations)
    x = b.x.cpu().numpy()
    nr = np.linalg.norm(ref.x, axis=1)
    assert np.all(np.linalg.norm(x - ref.x, axis=1) <= 1e-9 * np.maximum(nr, 1e-300) + 1e-12)


@pytest.mark.parametrize("M,K", [(128, 128), (224, 100), (200, 180)])
def test_batched_least_squares_beyond_shared_memory(M, K):
    rng = np.random.default_rng(M + K)
    P = 6
    b = rng.standard_normal((P, M, K))
    y = rng.standard_normal((P, M))
    s = gk.least_squares(b, y)
    for p in range(P):
        ref = oc.least_squares(b[p], y[p])
        np.testing.assert_allclose(s[p], ref, rtol=0, atol=1e-9 * max(1.0, np.abs(ref).max()))


def test_recover_cube_on_an_explicit_stream():
    c = _cube(P=4096, n=198)
    dic = Dictionary.per_pixel(c.basis, c.masks)
    cfg = SolverConfig(kappa=24, atoms_per_iter=4, time_limit=None)
    meas = c.y.reshape(512, 8, -1)
    ref_cube, ref_st = recover_cube(meas, dic, cfg, "gomp")
    s = torch.cuda.Stream()
    # keep the default stream busy so an unordered read would see stale results
    big = torch.empty(1 << 26, dtype=torch.float64, device="cuda")
    big.normal_()
    cube, st = recover_cube(meas, dic, cfg, "gomp", stream=s)
    np.testing.assert_array_equal(cube, ref_cube)
    assert (st.n_converged, st.total_iterations, st.n_failed) == (ref_st.n_converged, ref_st.total_iterations,
                                                                    ref_st.n_failed)
    np.testing.assert_array_equal(st.iterations, ref_st.iterations)
    # device input on the explicit stream
    dcube, dst = recover_cube(torch.as_tensor(meas, device="cuda"), dic, cfg, "gomp", stream=s)
    np.testing.assert_array_equal(dcube.cpu().numpy(), ref_cube)
    assert dst.total_iterations == ref_st.total_iterations


def test_recover_cube_sharded_single_process_equals_recover_cube():
    c = _cube(P=1200, n=154)
    dic = Dictionary.per_pixel(c.basis, c.masks)
    cfg = SolverConfig(kappa=22, mu=0.1, time_limit=None, max_iter=2000)
    meas = c.y.reshape(150, 8, -1)
    ref_cube, ref_st = recover_cube(meas, dic, cfg, "biht")
    (x0, x1), cube, summ = parallel.recover_cube_sharded(meas, dic, cfg, "biht")
    assert (x0, x1) == (0, 150)
    np.testing.assert_array_equal(cube, ref_cube)
    assert summ["n_pixels"] == 1200 and summ["total_iterations"] == ref_st.total_iterations
    assert summ["n_converged"] == ref_st.n_converged
