"""ctypes bindings of the C ABI in include/fpg.h (libfpg.so) and of the
corpus generators (libfpcorpus.so).

The product path is libfpg.so only; there is no CPU fallback.  If the
library is missing, loading fails loudly with instructions to build it.
"""
from __future__ import annotations

import ctypes
import os
from pathlib import Path

PKG = Path(__file__).resolve().parent
LIB_DIR = PKG / "lib"
LIBFPG = LIB_DIR / "libfpg.so"
LIBCORPUS = LIB_DIR / "libfpcorpus.so"

c_u8p = ctypes.POINTER(ctypes.c_uint8)
c_u32p = ctypes.POINTER(ctypes.c_uint32)
c_u64p = ctypes.POINTER(ctypes.c_uint64)


class FpgScheme(ctypes.Structure):
    _fields_ = [
        ("variant", ctypes.c_int32),
        ("width", ctypes.c_int32),
        ("bits_per_count", ctypes.c_int32),
        ("bits_per_position", ctypes.c_int32),
        ("nletters", ctypes.c_int32),
        ("letters", ctypes.c_uint8 * 64),
    ]


class FpgQueryOptions(ctypes.Structure):
    _fields_ = [
        ("metric", ctypes.c_int32),
        ("k", ctypes.c_int32),
        ("use_filter", ctypes.c_int32),
        ("length_prefilter", ctypes.c_int32),
        ("want_stats", ctypes.c_int32),
        ("exhaustive", ctypes.c_int32),
    ]


class FpgResult(ctypes.Structure):
    _fields_ = [
        ("nq", ctypes.c_uint64),
        ("total", ctypes.c_uint64),
        ("offsets", c_u64p),
        ("word_ids", c_u32p),
        ("stats", c_u64p),
    ]


# Every symbol include/fpg.h declares, with its ctypes signature.
FPG_SIGNATURES = {
    "fpg_last_error": (ctypes.c_char_p, []),
    "fpg_abi_version": (ctypes.c_int, []),
    "fpg_device_count": (ctypes.c_int, [ctypes.POINTER(ctypes.c_int)]),
    "fpg_letter_capacity": (ctypes.c_int, [ctypes.c_int32] * 4),
    "fpg_scheme_validate": (ctypes.c_int, [ctypes.POINTER(FpgScheme)]),
    "fpg_scheme_supports": (ctypes.c_int, [ctypes.POINTER(FpgScheme), ctypes.c_int32]),
    "fpg_dict_create": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint64,
                                       ctypes.POINTER(FpgScheme), ctypes.POINTER(ctypes.c_int32),
                                       ctypes.c_int32, ctypes.c_uint64,
                                       ctypes.POINTER(ctypes.c_void_p)]),
    "fpg_dict_create_from_text": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_uint64, ctypes.POINTER(FpgScheme),
                                                 ctypes.POINTER(ctypes.c_int32), ctypes.c_int32, ctypes.c_uint64,
                                                 ctypes.POINTER(ctypes.c_void_p)]),
    "fpg_byte_histogram": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int32, ctypes.c_void_p]),
    "fpg_dict_destroy": (ctypes.c_int, [ctypes.c_void_p]),
    "fpg_dict_size": (ctypes.c_int, [ctypes.c_void_p, c_u64p]),
    "fpg_dict_prints": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p]),
    "fpg_dict_build_seconds": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(ctypes.c_double)]),
    "fpg_dict_build_profile": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int32, ctypes.c_void_p, ctypes.c_int32,
                                              ctypes.POINTER(ctypes.c_int32)]),
    "fpg_build_fingerprints": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint64,
                                              ctypes.POINTER(FpgScheme), ctypes.c_int32,
                                              ctypes.c_void_p]),
    "fpg_query_batch": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                       ctypes.c_uint64, ctypes.POINTER(FpgQueryOptions),
                                       ctypes.POINTER(FpgResult)]),
    "fpg_result_free": (ctypes.c_int, [ctypes.POINTER(FpgResult)]),
    "fpg_batch_create": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(ctypes.c_void_p)]),
    "fpg_batch_destroy": (ctypes.c_int, [ctypes.c_void_p]),
    "fpg_batch_upload": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                        ctypes.c_uint64]),
    "fpg_batch_run": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(FpgQueryOptions)]),
    "fpg_batch_download": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(FpgResult)]),
    "fpg_batch_last_timing": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int32,
                                             ctypes.POINTER(ctypes.c_double),
                                             ctypes.POINTER(ctypes.c_double), c_u64p, c_u64p,
                                             c_u64p]),
    "fpg_batch_last_candidates": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int32, c_u64p]),
    "fpg_batch_last_verify": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int32, ctypes.POINTER(ctypes.c_double), c_u64p,
                                             ctypes.POINTER(ctypes.c_uint32), ctypes.POINTER(ctypes.c_double)]),
    "fpg_batch_last_scanned": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int32, c_u64p]),
    "fpg_batch_last_scanned_exact": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int32, c_u64p]),
    "fpg_batch_last_host_ms": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(ctypes.c_double),
                                              ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double)]),
    "fpg_batch_device_csr": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int32, ctypes.POINTER(ctypes.c_int32),
                                            c_u64p, ctypes.POINTER(ctypes.c_void_p),
                                            ctypes.POINTER(ctypes.c_void_p)]),
    "fpg_csr_merge_device": (ctypes.c_int, [ctypes.c_int32, ctypes.c_int32, ctypes.POINTER(ctypes.c_void_p),
                                            ctypes.POINTER(ctypes.c_void_p), ctypes.c_uint64, ctypes.c_void_p,
                                            ctypes.c_void_p, ctypes.c_void_p]),
    "fpg_dict_scan_shape": (ctypes.c_int, [ctypes.c_void_p, ctypes.POINTER(ctypes.c_int32),
                                           ctypes.POINTER(ctypes.c_int32)]),
}

FPG_OK, FPG_EINVAL, FPG_EUNSUPPORTED, FPG_ECUDA, FPG_ENOMEM = 0, -1, -2, -3, -4
FPG_ABI_VERSION = 3  # include/fpg.h

_fpg = None
_corpus = None


class FpgBuildStage(ctypes.Structure):
    _fields_ = [("name", ctypes.c_char * 24), ("ms", ctypes.c_double), ("bytes", ctypes.c_double)]


class FpgError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"fpg error {code}: {msg}")
        self.code = code


def load_fpg() -> ctypes.CDLL:
    """Loads libfpg.so (the CUDA product library).  Raises if absent."""
    global _fpg
    if _fpg is None:
        if not LIBFPG.exists():
            raise ImportError(
                f"{LIBFPG} is missing: the CUDA extension is not built. Run "
                "`python -c 'import __graft_entry__ as g; g.build()'` (nvcc, sm_100a).")
        lib = ctypes.CDLL(str(LIBFPG))
        for name, (res, args) in FPG_SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if lib.fpg_abi_version() != FPG_ABI_VERSION:
            raise ImportError(f"{LIBFPG} has ABI {lib.fpg_abi_version()}, these bindings expect "
                              f"{FPG_ABI_VERSION}: rebuild it (__graft_entry__.build())")
        _fpg = lib
    return _fpg


def check(code: int) -> None:
    if code != FPG_OK:
        msg = load_fpg().fpg_last_error().decode(errors="replace")
        if code == FPG_EINVAL:
            raise ValueError(msg)  # std::invalid_argument in the reference
        raise FpgError(code, msg)


def load_corpus() -> ctypes.CDLL:
    global _corpus
    if _corpus is None:
        if not LIBCORPUS.exists():
            raise ImportError(f"{LIBCORPUS} is missing; run __graft_entry__.build()")
        lib = ctypes.CDLL(str(LIBCORPUS))
        lib.fpc_max_len.restype = ctypes.c_int
        lib.fpc_max_len.argtypes = [ctypes.c_int]
        lib.fpc_dict_lengths.restype = ctypes.c_int64
        lib.fpc_dict_lengths.argtypes = [ctypes.c_int, ctypes.c_uint64, ctypes.c_uint64,
                                         ctypes.c_void_p, ctypes.c_int]
        lib.fpc_dict_fill.restype = ctypes.c_int
        lib.fpc_dict_fill.argtypes = [ctypes.c_int, ctypes.c_uint64, ctypes.c_uint64,
                                      ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int]
        lib.fpc_dict_lengths_at.restype = ctypes.c_int64
        lib.fpc_dict_lengths_at.argtypes = [ctypes.c_int, ctypes.c_uint64, ctypes.c_uint64,
                                            ctypes.c_uint64, ctypes.c_void_p, ctypes.c_int]
        lib.fpc_dict_fill_at.restype = ctypes.c_int
        lib.fpc_dict_fill_at.argtypes = [ctypes.c_int, ctypes.c_uint64, ctypes.c_uint64,
                                         ctypes.c_uint64, ctypes.c_void_p, ctypes.c_void_p,
                                         ctypes.c_int]
        lib.fpc_queries.restype = ctypes.c_int64
        lib.fpc_queries.argtypes = [ctypes.c_int, ctypes.c_uint64, ctypes.c_void_p,
                                    ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint64,
                                    ctypes.c_void_p, ctypes.c_uint64, ctypes.c_void_p]
        _corpus = lib
    return _corpus


def ptr(a):
    """Data pointer of a numpy array as c_void_p."""
    return ctypes.c_void_p(a.ctypes.data) if a is not None and a.size else ctypes.c_void_p(0)


def host_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1
