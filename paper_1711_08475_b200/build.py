"""In-tree build of the native libraries (no JIT cache: the .so files travel
with the repo snapshot to the GPU box).

  lib/libfpg.so       CUDA kernels + C ABI (include/fpg.h), sm_100a only
  lib/libfpcorpus.so  seeded config generators (host C)
"""
from __future__ import annotations

import os
import shutil
import subprocess
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB = PKG / "lib"

NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
              "-Xcompiler", "-fPIC", "-Xptxas", "-warn-spills"]


def _nvcc() -> str:
    for c in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if c and os.path.exists(c):
            return c
    raise RuntimeError("nvcc not found")


def _stale(target: Path, sources) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(Path(s).stat().st_mtime > t for s in sources)


def build_fpg(force: bool = False) -> Path:
    """Every csrc/*.cu compiled to an object in parallel (the K2 template
    instantiations live in their own translation units), then linked."""
    LIB.mkdir(exist_ok=True)
    out = LIB / "libfpg.so"
    units = sorted(CSRC.glob("*.cu"))
    srcs = units + sorted(CSRC.glob("*.cuh")) + sorted(CSRC.glob("*.h")) + [ROOT / "include" / "fpg.h"]
    if force or _stale(out, srcs):
        obj_dir = LIB / "obj"
        obj_dir.mkdir(exist_ok=True)
        dbg = ["-DFPG_DEBUG"] if os.environ.get("FPG_DEBUG") == "1" else []
        objs = [obj_dir / (u.stem + ".o") for u in units]
        procs = [subprocess.Popen([_nvcc(), *NVCC_FLAGS, *dbg, "-c", "-o", str(o), str(u)])
                 for u, o in zip(units, objs)]
        if any(pr.wait() != 0 for pr in procs):
            raise subprocess.CalledProcessError(1, "nvcc (see output above)")
        tmp = out.with_suffix(".so.tmp")
        subprocess.run([_nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", str(tmp),
                        *map(str, objs)], check=True)
        os.replace(tmp, out)
    return out


def build_corpus(force: bool = False) -> Path:
    LIB.mkdir(exist_ok=True)
    out = LIB / "libfpcorpus.so"
    src = CSRC / "corpus" / "fpcorpus.c"
    if force or _stale(out, [src, src.with_suffix(".h")]):
        subprocess.run(["gcc", "-O3", "-std=c11", "-fPIC", "-shared", "-pthread", "-o", str(out), str(src)],
                       check=True)
    return out


def build_all(force: bool = False) -> None:
    build_corpus(force)
    build_fpg(force)


if __name__ == "__main__":
    build_all(force=True)
