"""Build libhypercs_b200.so in-tree with nvcc for sm_100a.

    python -m paper_2401_14762_b200.build

The library is a plain C-ABI shared object (include/hypercs_b200.h) loaded by
ctypes; no torch headers are involved, so a rebuild takes seconds.
"""

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB = PKG / "libhypercs_b200.so"
# bounds-checked variant (shared-memory poison / canaries, device index
# assertions; hcs_common.cuh): select it with HCS_LIB=<path> for the tests
LIB_CHECKED = PKG / "libhypercs_b200_checked.so"

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-shared", "-Xcompiler", "-fPIC",
    "-I", str(ROOT / "include"),
]


def nvcc_path():
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found")


def sources():
    return sorted(str(p) for p in CSRC.glob("*.cu"))


def up_to_date(lib=LIB):
    if not lib.exists():
        return False
    t = lib.stat().st_mtime
    deps = list(CSRC.glob("*")) + list((ROOT / "include").glob("*.h"))
    return all(p.stat().st_mtime <= t for p in deps)


def build(force=False, verbose=False, checked=False):
    """Compile each translation unit in parallel (-c), then link the shared
    object (``checked``: the -DHCS_CHECKS variant, libhypercs_b200_checked.so)."""
    lib = LIB_CHECKED if checked else LIB
    if not force and up_to_date(lib):
        return lib
    from concurrent.futures import ThreadPoolExecutor
    import tempfile
    nvcc = nvcc_path()
    flags = [f for f in NVCC_FLAGS if f != "-shared"] + (["-DHCS_CHECKS"] if checked else [])
    with tempfile.TemporaryDirectory(prefix="hcs_build_") as tmp:
        jobs = [(src, str(Path(tmp) / (Path(src).stem + ".o"))) for src in sources()]

        def compile_one(job):
            cmd = [nvcc, *flags, "-c", "-o", job[1], job[0]]
            if verbose:
                print(" ".join(cmd))
            return subprocess.run(cmd, capture_output=True, text=True)

        with ThreadPoolExecutor(max_workers=min(len(jobs), os.cpu_count() or 1)) as ex:
            results = list(ex.map(compile_one, jobs))
        for res in results:
            if res.returncode != 0:
                raise RuntimeError(f"nvcc failed:\n{res.stdout}\n{res.stderr}")
        cmd = [nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", str(lib) + ".tmp",
               *(o for _, o in jobs)]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"nvcc link failed:\n{res.stdout}\n{res.stderr}")
    os.replace(str(lib) + ".tmp", lib)
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True, checked="--checked" in sys.argv))
