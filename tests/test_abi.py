"""The C-ABI library: built for sm_100a, loads without a GPU, exports exactly
what include/hypercs_b200.h declares (no compute calls here)."""

import ctypes
import re
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "hypercs_b200.h"


def declared_functions():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:int|size_t|const char\*)\s+(hcs_\w+)\s*\(", text, flags=re.M)))


@pytest.fixture(scope="module")
def lib_path():
    from paper_2401_14762_b200 import build
    return build.build()


def test_header_declares_the_boundary():
    names = declared_functions()
    for required in ("hcs_recover", "hcs_recover_status", "hcs_workspace_bytes", "hcs_least_squares",
                     "hcs_argmax_k", "hcs_soft_threshold", "hcs_residual_delta", "hcs_lipschitz",
                     "hcs_psnr_partials", "hcs_last_error", "hcs_abi_version", "hcs_dmma_peak_tflops"):
        assert required in names


def test_library_exports_every_declared_symbol(lib_path):
    lib = ctypes.CDLL(str(lib_path))
    for name in declared_functions():
        assert hasattr(lib, name), name
    from paper_2401_14762_b200 import _native
    assert set(_native.EXPORTS) <= set(declared_functions())


def test_library_is_sm100a(lib_path):
    out = subprocess.run(["cuobjdump", "--list-elf", str(lib_path)], capture_output=True, text=True)
    assert out.returncode == 0
    assert "sm_100a" in out.stdout


def test_sass_uses_fp64_tensor_cores(lib_path):
    out = subprocess.run(["cuobjdump", "-sass", str(lib_path)], capture_output=True, text=True).stdout
    assert "DMMA.8x8x4" in out          # FP64 mma.sync in the GEMM / least-squares paths
    assert "LDGSTS" in out              # cp.async gathers


def test_host_only_entry_points(lib_path):
    from paper_2401_14762_b200 import _native
    lib = _native.load(lib_path)
    assert lib.hcs_abi_version() == 101
    # workspace sizing needs no device for the convex solvers
    assert lib.hcs_workspace_bytes(0, 1000, 198, 79) >= 2 * 208 * 208 * 8
    # argument validation happens before any device work
    prm = _native.HcsParams(lam=0.1, mu=0.1, alpha=1.8, epsilon=1e-8, kappa=30, atoms_per_iter=0, max_iter=10)
    st = _native.HcsStats()
    code = lib.hcs_recover(4, 10, 224, 90, None, None, None, prm, None, st, None, 0, None)
    assert code == _native.HCS_EINVAL
    assert b"kappa" in lib.hcs_last_error() or b"stats" in lib.hcs_last_error()
    code = lib.hcs_argmax_k(1, 8, None, 9, None, None)
    assert code == _native.HCS_EINVAL and b"k must be in [1, 8]" in lib.hcs_last_error()
