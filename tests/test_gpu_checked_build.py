"""Memory-safety evidence without compute-sanitizer (closed on this GPU pool).

The bounds-checked library (libhypercs_b200_checked.so, -DHCS_CHECKS; see
hcs_common.cuh) poisons every CTA's dynamic shared memory with a NaN bit
pattern at kernel entry (reads of unwritten shared memory turn results
non-finite), verifies a canary block after the dynamic region at exit
(out-of-bounds shared stores) and asserts the data-dependent bounds
(least-squares sizes vs their buffers, scratch slots).  These tests run the
small-case driver over every kernel family and the oracle-parity suite
against the checked library in a subprocess, check a deliberate overrun is
caught (positive control), and check that hcs_recover never writes outside
its output arrays (guard zones, regular build).
"""

import ctypes
import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from paper_2401_14762_b200 import _native as nat  # noqa: E402
from paper_2401_14762_b200 import build, synth  # noqa: E402

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


@pytest.fixture(scope="module")
def checked_lib():
    lib = build.LIB_CHECKED
    if not lib.exists():
        build.build(checked=True)
    return str(lib)


def _run(args, lib, extra_env=None, timeout=900):
    env = dict(os.environ, HCS_LIB=lib, **(extra_env or {}))
    return subprocess.run([sys.executable, *args], cwd=ROOT, env=env, capture_output=True, text=True,
                          timeout=timeout)


def test_checked_library_runs_every_kernel_family(checked_lib):
    r = _run([str(ROOT / "tools" / "sanitize_cases.py")], checked_lib)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert "ok input side" in r.stdout
    code = _run(["-c", "from paper_2401_14762_b200 import _native as n; print(n.load().hcs_checked_build())"],
                checked_lib)
    assert code.stdout.strip() == "1"


def test_checked_library_passes_oracle_parity(checked_lib):
    r = _run(["-m", "pytest", "-q", "-x", "-p", "no:cacheprovider", "tests/test_gpu_parity.py",
              "tests/test_gpu_api.py", "tests/test_gpu_selection.py"], checked_lib, timeout=1800)
    assert r.returncode == 0, r.stdout[-3000:]


def test_checked_library_catches_a_shared_overrun(checked_lib):
    """Positive control: HCS_CHECK_SELFTEST=1 makes the warp gOMP kernel flip
    a byte past its shared region; the canary check must report it."""
    code = ("import torch, numpy as np\n"
            "from paper_2401_14762_b200 import synth\n"
            "from paper_2401_14762_b200.solvers import SolverConfig, solve_batch\n"
            "c = synth.generate(4, 8, 224, seed=1)\n"
            "d = torch.device('cuda')\n"
            "try:\n"
            "    solve_batch('gomp', torch.as_tensor(c.y, device=d), torch.as_tensor(c.masks, device=d),\n"
            "                torch.as_tensor(c.basis, device=d), SolverConfig(kappa=27, time_limit=None))\n"
            "    print('NOT CAUGHT')\n"
            "except RuntimeError as e:\n"
            "    print('CAUGHT', e)\n")
    r = _run(["-c", code], checked_lib, {"HCS_CHECK_SELFTEST": "1"})
    assert "CAUGHT" in r.stdout and "canary" in r.stdout, r.stdout + r.stderr


@pytest.mark.parametrize("algo", [0, 1, 2, 3, 4])
def test_outputs_stay_inside_their_arrays(algo):
    """Guard zones around x_out and every stats array stay untouched."""
    lib = nat.load()
    c = synth.generate(8, 8, 224, seed=2)
    P, m = c.y.shape
    n = c.n
    G = 64
    dev = torch.device("cuda")

    def guarded(count, dtype, fill):
        t = torch.full((count + 2 * G,), fill, dtype=dtype, device=dev)
        return t, t[G:G + count]

    xg, x = guarded(P * n, torch.float64, 12345.0)
    itg, it = guarded(P, torch.int32, -7)
    cvg, cv = guarded(P, torch.uint8, 77)
    fdg, fd = guarded(P, torch.float64, 12345.0)
    fag, fa = guarded(P, torch.int32, -7)
    gpg, gp = guarded(P, torch.float64, 12345.0)
    lpg, lp = guarded(P, torch.float64, 12345.0)
    elg, el = guarded(P, torch.float64, 12345.0)
    wkg, wk = guarded(P, torch.float64, 12345.0)
    st = nat.HcsStats(iterations=it.data_ptr(), converged=cv.data_ptr(), final_delta=fd.data_ptr(),
                      failed_at=fa.data_ptr(), admm_gap=gp.data_ptr(), lipschitz=lp.data_ptr(),
                      elapsed=el.data_ptr(), work=wk.data_ptr())
    prm = nat.HcsParams(lam=0.1, mu=0.1, alpha=1.8, epsilon=1e-8, kappa=27, atoms_per_iter=0, max_iter=300)
    wsb = lib.hcs_workspace_bytes(algo, P, n, m)
    wsg, ws = guarded(wsb, torch.uint8, 0xA5)
    yd, md, bd = (torch.as_tensor(a, device=dev) for a in (c.y, c.masks, c.basis))
    assert lib.hcs_recover(algo, P, n, m, bd.data_ptr(), yd.data_ptr(), md.data_ptr(), prm, x.data_ptr(), st,
                           ws.data_ptr(), wsb, None) == nat.HCS_OK
    assert lib.hcs_recover_status(ws.data_ptr(), None) == nat.HCS_OK
    torch.cuda.synchronize()
    for g in (xg, itg, cvg, fdg, fag, gpg, lpg, elg, wkg, wsg):
        head, tail = g[:G].cpu().numpy(), g[-G:].cpu().numpy()
        assert np.all(head == head[0]) and np.all(tail == head[0])
    assert np.all(it.cpu().numpy() >= 0)
