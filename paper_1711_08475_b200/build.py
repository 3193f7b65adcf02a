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
              "-Xcompiler", "-fPIC", "-shared", "-Xptxas", "-warn-spills"]


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
    LIB.mkdir(exist_ok=True)
    out = LIB / "libfpg.so"
    srcs = sorted(CSRC.glob("*.cu")) + sorted(CSRC.glob("*.cuh")) + [ROOT / "include" / "fpg.h"]
    if force or _stale(out, srcs):
        tmp = out.with_suffix(".so.tmp")
        dbg = ["-DFPG_DEBUG"] if os.environ.get("FPG_DEBUG") == "1" else []
        cmd = [_nvcc(), *NVCC_FLAGS, *dbg, "-o", str(tmp), str(CSRC / "fpg_api.cu")]
        subprocess.run(cmd, check=True)
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
