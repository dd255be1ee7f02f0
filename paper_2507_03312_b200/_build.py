"""Build the native library libmpx_b200.so in-tree (nvcc, sm_100a only).

The .so lands in paper_2507_03312_b200/lib/ so it travels with the repo to
the GPU box (it is git-ignored, not gpurun-ignored).  Objects are cached in
build/ and rebuilt when a source or header is newer.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
INCLUDE = ROOT / "include"
OBJ = ROOT / "build" / "obj"
LIB = PKG / "lib" / "libmpx_b200.so"

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
# IEEE-exact arithmetic is part of the numerics contract: no FTZ, correctly
# rounded div/sqrt.  Kernels that need no contraction use __f*_rn intrinsics.
NVCC_FLAGS = ARCH + [
    "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
    "-ftz=false", "-prec-div=true", "-prec-sqrt=true",
    "--expt-relaxed-constexpr", "-I", str(INCLUDE),
]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found: cannot build libmpx_b200.so")


def _sources() -> list[Path]:
    return sorted(CSRC.glob("*.cu"))


def _headers() -> list[Path]:
    return sorted(CSRC.glob("*.cuh")) + sorted(INCLUDE.glob("*.h"))


def _stale(target: Path, deps: list[Path]) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps)


def build(verbose: bool = False, force: bool = False, defines: tuple = (), out: Path | None = None) -> Path:
    """defines: extra -D macros for an instrumented variant (objects in
    build/obj-<tag>, library at `out`); the product build has none."""
    obj_dir = OBJ if not defines else OBJ.parent / ("obj-" + "-".join(d.lower() for d in defines))
    lib = LIB if out is None else Path(out)
    obj_dir.mkdir(parents=True, exist_ok=True)
    lib.parent.mkdir(parents=True, exist_ok=True)
    flags = NVCC_FLAGS + [f"-D{d}" for d in defines]
    headers = _headers()
    cc = nvcc()
    jobs = []
    objs = []
    for src in _sources():
        obj = obj_dir / (src.stem + ".o")
        objs.append(obj)
        if force or _stale(obj, [src] + headers):
            jobs.append([cc, *flags, "-c", str(src), "-o", str(obj)])

    def run(cmd):
        if verbose:
            print(" ".join(cmd), flush=True)
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed:\n{' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
        return r

    with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        list(ex.map(run, jobs))
    if force or jobs or _stale(lib, objs):
        run([cc, *ARCH, "-shared", "-o", str(lib), *map(str, objs), "-ldl"])
    return lib


if __name__ == "__main__":
    # python _build.py [-v] [-f] [-DNAME ... -o out.so]   (instrumented variants)
    defs = tuple(a[2:] for a in sys.argv[1:] if a.startswith("-D"))
    out = sys.argv[sys.argv.index("-o") + 1] if "-o" in sys.argv else None
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv, defines=defs, out=out))
