"""Python bindings of the CPU checkers.  TEST INFRASTRUCTURE ONLY.

* ``Oracle``    -> oracle/libfp_oracle.so, the C restatement (fp_oracle.c)
* ``Reference`` -> oracle/_ref/libfpref.so, the reference's own headers
                   compiled behind ref_driver.cpp (absent if never built)

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs may
import this module; the product (paper_1711_08475_b200, libfpg.so) never does.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ORACLE_SO = HERE / "libfp_oracle.so"
REF_SO = HERE / "_ref" / "libfpref.so"

vp = ctypes.c_void_p


class OScheme(ctypes.Structure):
    _fields_ = [("variant", ctypes.c_int), ("width", ctypes.c_int), ("bits_per_count", ctypes.c_int),
                ("bits_per_position", ctypes.c_int), ("nletters", ctypes.c_int),
                ("letters", ctypes.c_uint8 * 64)]


def _p(a):
    return vp(a.ctypes.data) if a is not None and a.size else vp(0)


def build_oracle() -> None:
    subprocess.run(["make", "-s", "-C", str(HERE)], check=True)


def pack(words):
    bs = [w.encode("latin-1") if isinstance(w, str) else bytes(w) for w in words]
    offs = np.zeros(len(bs) + 1, np.uint64)
    if bs:
        offs[1:] = np.cumsum([len(b) for b in bs])
    blob = np.frombuffer(b"".join(bs), np.uint8).copy() if bs else np.zeros(0, np.uint8)
    return blob, offs


def oscheme(variant: int, letters, width: int = 16, b: int = 2, p: int = 3) -> OScheme:
    s = OScheme()
    s.variant, s.width, s.bits_per_count, s.bits_per_position = int(variant), width, b, p
    lb = letters.encode("latin-1") if isinstance(letters, str) else bytes(letters)
    s.nletters = len(lb)
    for i, c in enumerate(lb):
        s.letters[i] = c
    return s


class Oracle:
    """C restatement of the reference path, generalised to W in {16,32,64}."""

    def __init__(self):
        if not ORACLE_SO.exists():
            build_oracle()
        L = ctypes.CDLL(str(ORACLE_SO))
        L.fpo_build.restype = ctypes.c_uint64
        L.fpo_build.argtypes = [vp, ctypes.c_size_t, ctypes.POINTER(OScheme)]
        L.fpo_build_many.argtypes = [vp, vp, ctypes.c_uint64, ctypes.POINTER(OScheme), vp]
        L.fpo_distance.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.POINTER(OScheme)]
        L.fpo_can_reject.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int, ctypes.POINTER(OScheme)]
        L.fpo_render.argtypes = [ctypes.c_uint64, ctypes.POINTER(OScheme), ctypes.c_char_p]
        L.fpo_letter_capacity.argtypes = [ctypes.c_int] * 4
        L.fpo_scheme_check.argtypes = [ctypes.POINTER(OScheme)]
        L.fpo_select_letters.argtypes = [vp, ctypes.c_uint64, ctypes.c_int, ctypes.c_int, ctypes.c_char_p]
        for f in ("fpo_hamming_bounded", "fpo_levenshtein_bounded"):
            getattr(L, f).argtypes = [ctypes.c_char_p, ctypes.c_size_t, ctypes.c_char_p, ctypes.c_size_t, ctypes.c_int]
        for f in ("fpo_hamming_full", "fpo_levenshtein_full"):
            getattr(L, f).argtypes = [ctypes.c_char_p, ctypes.c_size_t, ctypes.c_char_p, ctypes.c_size_t]
        L.fpo_query_batch.argtypes = [vp, vp, ctypes.c_uint64, vp, vp, ctypes.c_uint64,
                                      ctypes.POINTER(OScheme), ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                      ctypes.c_int, ctypes.c_int, vp, vp,
                                      ctypes.POINTER(ctypes.POINTER(ctypes.c_uint32)),
                                      ctypes.POINTER(ctypes.c_uint64)]
        L.fpo_naive_scan_batch.argtypes = [vp, vp, ctypes.c_uint64, vp, vp, ctypes.c_uint64,
                                           ctypes.c_int, ctypes.c_int, ctypes.c_int, vp,
                                           ctypes.POINTER(ctypes.POINTER(ctypes.c_uint32)),
                                           ctypes.POINTER(ctypes.c_uint64)]
        L.fpo_free.argtypes = [vp]
        self.L = L

    def build(self, s, sch: OScheme) -> int:
        b = s.encode("latin-1") if isinstance(s, str) else bytes(s)
        return int(self.L.fpo_build(ctypes.c_char_p(b), len(b), ctypes.byref(sch)))

    def build_many(self, blob, offs, sch: OScheme) -> np.ndarray:
        n = len(offs) - 1
        out = np.zeros(max(n, 1), np.uint64)
        self.L.fpo_build_many(_p(blob), _p(offs), n, ctypes.byref(sch), _p(out))
        return out[:n]

    def distance(self, a: int, b: int, sch: OScheme) -> int:
        return self.L.fpo_distance(a, b, ctypes.byref(sch))

    def can_reject(self, a, b, k, sch) -> bool:
        return bool(self.L.fpo_can_reject(a, b, k, ctypes.byref(sch)))

    def render(self, f: int, sch: OScheme) -> str:
        buf = ctypes.create_string_buffer(160)
        self.L.fpo_render(f, ctypes.byref(sch), buf)
        return buf.value.decode()

    def letter_capacity(self, v, w, b=2, p=3) -> int:
        return self.L.fpo_letter_capacity(v, w, b, p)

    def scheme_ok(self, sch) -> bool:
        return self.L.fpo_scheme_check(ctypes.byref(sch)) == 0

    def select_letters(self, blob, count, strategy) -> bytes | None:
        buf = ctypes.create_string_buffer(256)
        r = self.L.fpo_select_letters(_p(blob), blob.size, count, strategy, buf)
        return None if r < 0 else buf.raw[:r]

    def _verify(self, f, a, b, k=None):
        a = a.encode("latin-1") if isinstance(a, str) else bytes(a)
        b = b.encode("latin-1") if isinstance(b, str) else bytes(b)
        args = [a, len(a), b, len(b)] + ([] if k is None else [k])
        return getattr(self.L, f)(*args)

    def hamming_bounded(self, a, b, k):
        return self._verify("fpo_hamming_bounded", a, b, k)

    def levenshtein_bounded(self, a, b, k):
        return self._verify("fpo_levenshtein_bounded", a, b, k)

    def levenshtein_full(self, a, b):
        return self._verify("fpo_levenshtein_full", a, b)

    def hamming_full(self, a, b):
        return self._verify("fpo_hamming_full", a, b)

    def query_batch(self, dblob, doffs, qblob, qoffs, sch: OScheme, metric, k=1, use_filter=True,
                    length_prefilter=False, threads=None):
        """Returns (offsets[nq+1], ids, stats[nq,5])."""
        nd, nq = len(doffs) - 1, len(qoffs) - 1
        offsets = np.zeros(nq + 1, np.uint64)
        stats = np.zeros((max(nq, 1), 5), np.uint64)
        ids = ctypes.POINTER(ctypes.c_uint32)()
        total = ctypes.c_uint64()
        r = self.L.fpo_query_batch(_p(dblob), _p(doffs), nd, _p(qblob), _p(qoffs), nq, ctypes.byref(sch),
                                   int(metric), k, int(use_filter), int(length_prefilter),
                                   threads or os.cpu_count(), _p(offsets), _p(stats), ctypes.byref(ids),
                                   ctypes.byref(total))
        if r != 0:
            raise ValueError("scheme does not filter for this metric")
        out = np.ctypeslib.as_array(ids, shape=(max(total.value, 1),))[: total.value].copy()
        self.L.fpo_free(ctypes.cast(ids, vp))
        return offsets, out, stats[:nq]

    def naive_scan_batch(self, dblob, doffs, qblob, qoffs, metric, k=1, threads=None):
        nd, nq = len(doffs) - 1, len(qoffs) - 1
        offsets = np.zeros(nq + 1, np.uint64)
        ids = ctypes.POINTER(ctypes.c_uint32)()
        total = ctypes.c_uint64()
        self.L.fpo_naive_scan_batch(_p(dblob), _p(doffs), nd, _p(qblob), _p(qoffs), nq, int(metric), k,
                                    threads or os.cpu_count(), _p(offsets), ctypes.byref(ids),
                                    ctypes.byref(total))
        out = np.ctypeslib.as_array(ids, shape=(max(total.value, 1),))[: total.value].copy()
        self.L.fpo_free(ctypes.cast(ids, vp))
        return offsets, out


class Reference:
    """The reference's own header-only library (W=16), via oracle/_ref."""

    @staticmethod
    def available() -> bool:
        return REF_SO.exists()

    def __init__(self):
        if not REF_SO.exists():
            raise FileNotFoundError(f"{REF_SO} not built (reference tree absent)")
        L = ctypes.CDLL(str(REF_SO))
        L.fpr_scheme_check.argtypes = [ctypes.c_int, ctypes.c_char_p, ctypes.c_int, ctypes.c_int, ctypes.c_int]
        L.fpr_letter_capacity.argtypes = [ctypes.c_int] * 3
        L.fpr_select_letters.argtypes = [vp, ctypes.c_uint64, ctypes.c_int, ctypes.c_int, ctypes.c_char_p]
        L.fpr_build_many.argtypes = [vp, vp, ctypes.c_uint64, ctypes.c_int, ctypes.c_char_p, ctypes.c_int,
                                     ctypes.c_int, ctypes.c_int, vp]
        L.fpr_distance_table.argtypes = [ctypes.c_int, ctypes.c_char_p, ctypes.c_int, ctypes.c_int,
                                         ctypes.c_int, vp]
        L.fpr_render.argtypes = [ctypes.c_uint16, ctypes.c_int, ctypes.c_char_p, ctypes.c_int, ctypes.c_int,
                                 ctypes.c_int, ctypes.c_char_p]
        for f in ("fpr_hamming_bounded", "fpr_levenshtein_bounded"):
            getattr(L, f).argtypes = [ctypes.c_char_p, ctypes.c_size_t, ctypes.c_char_p, ctypes.c_size_t, ctypes.c_int]
        L.fpr_levenshtein_full.argtypes = [ctypes.c_char_p, ctypes.c_size_t, ctypes.c_char_p, ctypes.c_size_t]
        L.fpr_dict_create.restype = vp
        L.fpr_dict_create.argtypes = [vp, vp, ctypes.c_uint64, ctypes.c_int, ctypes.c_char_p, ctypes.c_int,
                                      ctypes.c_int, ctypes.c_int]
        L.fpr_dict_destroy.argtypes = [vp]
        L.fpr_query_batch.argtypes = [vp, vp, vp, ctypes.c_uint64, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                      ctypes.c_int, ctypes.c_int, vp, vp,
                                      ctypes.POINTER(ctypes.POINTER(ctypes.c_uint32)),
                                      ctypes.POINTER(ctypes.c_uint64)]
        L.fpr_free.argtypes = [vp]
        self.L = L

    @staticmethod
    def _lb(letters):
        return letters.encode("latin-1") if isinstance(letters, str) else bytes(letters)

    def build_many(self, blob, offs, variant, letters, b=2, p=3) -> np.ndarray:
        n = len(offs) - 1
        out = np.zeros(max(n, 1), np.uint16)
        lb = self._lb(letters)
        r = self.L.fpr_build_many(_p(blob), _p(offs), n, variant, lb, len(lb), b, p, _p(out))
        if r:
            raise ValueError("invalid scheme")
        return out[:n]

    def distance_table(self, variant, letters, b=2, p=3) -> np.ndarray:
        out = np.zeros(65536, np.uint8)
        lb = self._lb(letters)
        if self.L.fpr_distance_table(variant, lb, len(lb), b, p, _p(out)):
            raise ValueError("invalid scheme")
        return out

    def render(self, f, variant, letters, b=2, p=3) -> str:
        buf = ctypes.create_string_buffer(64)
        lb = self._lb(letters)
        self.L.fpr_render(f, variant, lb, len(lb), b, p, buf)
        return buf.value.decode()

    def scheme_ok(self, variant, letters, b=2, p=3) -> bool:
        lb = self._lb(letters)
        return self.L.fpr_scheme_check(variant, lb, len(lb), b, p) == 0

    def letter_capacity(self, v, b=2, p=3) -> int:
        return self.L.fpr_letter_capacity(v, b, p)

    def select_letters(self, blob, count, strategy) -> bytes | None:
        buf = ctypes.create_string_buffer(256)
        r = self.L.fpr_select_letters(_p(blob), blob.size, count, strategy, buf)
        return None if r < 0 else buf.raw[:r]

    def hamming_bounded(self, a, b, k):
        a, b = self._lb(a), self._lb(b)
        return self.L.fpr_hamming_bounded(a, len(a), b, len(b), k)

    def levenshtein_bounded(self, a, b, k):
        a, b = self._lb(a), self._lb(b)
        return self.L.fpr_levenshtein_bounded(a, len(a), b, len(b), k)

    def levenshtein_full(self, a, b):
        a, b = self._lb(a), self._lb(b)
        return self.L.fpr_levenshtein_full(a, len(a), b, len(b))

    def dictionary(self, dblob, doffs, variant, letters, b=2, p=3):
        lb = self._lb(letters)
        h = self.L.fpr_dict_create(_p(dblob), _p(doffs), len(doffs) - 1, variant, lb, len(lb), b, p)
        if not h:
            raise ValueError("invalid scheme")
        return RefDict(self, h)


class RefDict:
    def __init__(self, ref: Reference, h):
        self.ref, self.h = ref, h

    def query_batch(self, qblob, qoffs, metric, k=1, use_filter=True, length_prefilter=False, threads=None):
        nq = len(qoffs) - 1
        offsets = np.zeros(nq + 1, np.uint64)
        stats = np.zeros((max(nq, 1), 5), np.uint64)
        ids = ctypes.POINTER(ctypes.c_uint32)()
        total = ctypes.c_uint64()
        r = self.ref.L.fpr_query_batch(self.h, _p(qblob), _p(qoffs), nq, int(metric), k, int(use_filter),
                                       int(length_prefilter), threads or os.cpu_count(), _p(offsets),
                                       _p(stats), ctypes.byref(ids), ctypes.byref(total))
        if r != 0:
            raise ValueError("scheme does not filter for this metric")
        out = np.ctypeslib.as_array(ids, shape=(max(total.value, 1),))[: total.value].copy()
        self.ref.L.fpr_free(ctypes.cast(ids, vp))
        return offsets, out, stats[:nq]

    def close(self):
        if self.h:
            self.ref.L.fpr_dict_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
