"""Build the CUDA library in-tree (the .so travels to the GPU box with gpurun).

    python -m paper_1303_7425_b200.build        # or __graft_entry__.build()

Produces paper_1303_7425_b200/lib/libpolymul_b200.so for sm_100a only.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
LIBDIR = PKG / "lib"
LIB = LIBDIR / "libpolymul_b200.so"
# device-side bounds assertions (-DPGPU_CHECKED): the checked build the GPU
# tests run every path through (tests/test_gpu_checked.py)
LIB_CHECKED = LIBDIR / "libpolymul_b200_checked.so"
ROOT = PKG.parent

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-shared",
    "--expt-relaxed-constexpr",
    "-Xptxas", "-warn-spills",
]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found: the CUDA library cannot be built")


def sources() -> list:
    return sorted(CSRC.glob("*.cu")) + sorted(CSRC.glob("*.cuh")) + sorted(CSRC.glob("*.inc")) + [
        ROOT / "include" / "polymul_b200.h"]


def stale(lib: Path = LIB) -> bool:
    if not lib.exists():
        return True
    t = lib.stat().st_mtime
    return any(s.stat().st_mtime > t for s in sources())


def build(force: bool = False, verbose: bool = False, out: Path | None = None,
          defines: tuple = ()) -> Path:
    if out is None and not force and not stale():
        return LIB
    LIBDIR.mkdir(exist_ok=True)
    target = Path(out) if out else LIB
    tmp = target.with_suffix(".so.tmp")
    cmd = [nvcc(), *NVCC_FLAGS, *[f"-D{d}" for d in defines], "-I", str(ROOT / "include"),
           str(CSRC / "polymul_b200.cu"), "-o", str(tmp)]
    if verbose:
        print(" ".join(cmd), flush=True)
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed ({res.returncode}):\n{res.stdout}\n{res.stderr}")
    if verbose and (res.stdout or res.stderr):
        print(res.stdout, res.stderr, file=sys.stderr)
    os.replace(tmp, target)
    return target


def build_checked(force: bool = False, verbose: bool = False) -> Path:
    """The checked library (device bounds assertions); same sources."""
    if not force and not stale(LIB_CHECKED):
        return LIB_CHECKED
    return build(force=True, verbose=verbose, out=LIB_CHECKED, defines=("PGPU_CHECKED",))


def build_pylimbs(force: bool = False) -> Path:
    """The CPython marshaling helper (csrc/pylimbs.c), built with gcc in-tree."""
    import sysconfig
    src = CSRC / "pylimbs.c"
    out = LIBDIR / ("_pylimbs" + sysconfig.get_config_var("EXT_SUFFIX"))
    if out.exists() and not force and out.stat().st_mtime >= src.stat().st_mtime:
        return out
    LIBDIR.mkdir(exist_ok=True)
    cc = shutil.which("gcc") or shutil.which("cc")
    if cc is None:
        raise RuntimeError("gcc not found: cannot build the marshaling helper")
    tmp = out.with_suffix(".tmp")
    cmd = [cc, "-O2", "-shared", "-fPIC", "-I", sysconfig.get_paths()["include"], str(src), "-o", str(tmp)]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"gcc failed ({res.returncode}):\n{res.stdout}\n{res.stderr}")
    os.replace(tmp, out)
    return out


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
    print(build_checked(force="--force" in sys.argv))
    print(build_pylimbs(force="--force" in sys.argv))
