import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs libfpg.so kernels)")
    config.addinivalue_line("markers", "slow: long-running")


def gpu_available() -> bool:
    try:
        from paper_1711_08475_b200._lib import load_fpg
        import ctypes
        n = ctypes.c_int(0)
        return load_fpg().fpg_device_count(ctypes.byref(n)) == 0 and n.value > 0
    except Exception:
        return False


@pytest.fixture(params=["exact-auto", "exact-forced"])
def exact_path(request, monkeypatch):
    """Runs a test twice: with K2's exact short-word Hamming path at its
    default work threshold (small test batches then stay on the sig' path),
    and forced on for every eligible tile (FPG_EXACT_MIN=0)."""
    if request.param == "exact-forced":
        monkeypatch.setenv("FPG_EXACT_MIN", "0")
    else:
        monkeypatch.delenv("FPG_EXACT_MIN", raising=False)
    return request.param


@pytest.fixture(scope="session")
def oracle():
    from oracle.oracle import Oracle
    return Oracle()


@pytest.fixture(scope="session")
def reference():
    from oracle.oracle import Reference
    if not Reference.available():
        pytest.skip("oracle/_ref not built (reference tree absent when building)")
    return Reference()


def build_api_check(tmp_dir: Path) -> Path:
    """Compiles tests/cpp/api_check.cpp against include/fingerprints/b200.hpp
    and links libfpg.so (the C++ drop-in surface)."""
    import shutil
    import subprocess

    from paper_1711_08475_b200._lib import LIBFPG

    cxx = shutil.which("g++")
    if not cxx:
        pytest.skip("g++ not available")
    exe = tmp_dir / "api_check"
    subprocess.run([cxx, "-std=c++20", "-O1", "-Wall", "-Werror", f"-I{ROOT / 'include'}",
                    str(ROOT / "tests" / "cpp" / "api_check.cpp"), f"-L{LIBFPG.parent}", "-lfpg",
                    f"-Wl,-rpath,{LIBFPG.parent}", "-o", str(exe)], check=True)
    return exe


REF_INCLUDE = Path("/root/reference/proj/include")
API_CHECK_REF_BIN = ROOT / "tests" / "cpp" / "_bin" / "api_check_ref"


def build_api_check_ref(out: Path = API_CHECK_REF_BIN) -> Path:
    """Compiles tests/cpp/api_check_ref.cpp: the reference's own headers
    (corpus / dictionary / reference.hpp, from /root/reference) and
    include/fingerprints/b200_ref.hpp in one translation unit, linked with
    libfpg.so.  Needs the reference tree (this container); __graft_entry__.build()
    leaves the binary in tests/cpp/_bin/ so it travels to the GPU box."""
    import shutil
    import subprocess

    from paper_1711_08475_b200._lib import LIBFPG

    cxx = shutil.which("g++")
    if not cxx or not (REF_INCLUDE / "fingerprints" / "dictionary.hpp").exists():
        raise FileNotFoundError("g++ or the reference headers are missing")
    out.parent.mkdir(parents=True, exist_ok=True)
    subprocess.run([cxx, "-std=c++20", "-O2", "-Wall", "-Werror", f"-I{REF_INCLUDE}", f"-I{ROOT / 'include'}",
                    str(ROOT / "tests" / "cpp" / "api_check_ref.cpp"), f"-L{LIBFPG.parent}", "-lfpg",
                    "-Wl,-rpath,$ORIGIN/../../../paper_1711_08475_b200/lib", f"-Wl,-rpath,{LIBFPG.parent}",
                    "-o", str(out)], check=True)
    return out
