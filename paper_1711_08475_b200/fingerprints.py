"""Host-side mirror of the reference's fingerprint / matching API, on the GPU.

Names, argument meaning and error behaviour follow the reference C++ library
(/root/reference/proj/include/fingerprints/): ``LetterSet``, ``Scheme``,
``Fingerprint``, ``build``, ``render``, ``QueryOptions``, ``QueryStats`` and
the dictionary with ``query`` / ``query_into``.  Every fingerprint, filter and
verification runs in libfpg.so (CUDA, sm_100a) through the C ABI of
include/fpg.h; this module only marshals arguments.  Invalid arguments raise
``ValueError`` where the reference throws ``std::invalid_argument``.

The dictionary class is ``GpuFingerprintedDictionary``; it
has the reference's method set plus ``query_batch``.  Schemes gain a width
``W`` in {16, 32, 64} (the reference fixes 16, fingerprint.hpp:31).
"""
from __future__ import annotations

import ctypes
import weakref
from dataclasses import dataclass
from enum import IntEnum
from typing import Iterable, Sequence

import numpy as np

from . import _lib
from ._lib import FpgQueryOptions, FpgResult, FpgScheme, check, load_fpg, ptr


class Variant(IntEnum):  # fingerprint.hpp:14
    Occurrence = 0
    OccurrenceHalved = 1
    Count = 2
    Position = 3


class Metric(IntEnum):  # fingerprint.hpp:15
    Hamming = 0
    Levenshtein = 1


class LetterStrategy(IntEnum):  # letter_model.hpp:47
    Common = 0
    Mixed = 1
    Rare = 2


def variant_supports(v: Variant, m: Metric) -> bool:
    """fingerprint.hpp:36-38: halved / position filter Hamming only."""
    return m == Metric.Hamming or v in (Variant.Occurrence, Variant.Count)


def _as_bytes(s) -> bytes:
    return s.encode("latin-1") if isinstance(s, str) else bytes(s)


def pack_strings(words: Iterable) -> tuple[np.ndarray, np.ndarray]:
    """Strings -> (byte blob uint8, offsets uint64 of length n+1)."""
    bs = [_as_bytes(w) for w in words]
    offsets = np.zeros(len(bs) + 1, dtype=np.uint64)
    if bs:
        offsets[1:] = np.cumsum([len(b) for b in bs], dtype=np.uint64)
    blob = np.frombuffer(b"".join(bs), dtype=np.uint8).copy() if bs else np.zeros(0, np.uint8)
    return blob, offsets


# ---------------------------------------------------------------- letters

class SymbolFrequencyTable:
    """letter_model.hpp:15-31: per-byte counts of a corpus."""

    def __init__(self):
        self.counts = np.zeros(256, dtype=np.uint64)
        self.total = 0

    def alphabet_size(self) -> int:
        return int(np.count_nonzero(self.counts))

    def add(self, corpus) -> None:
        data = corpus if isinstance(corpus, np.ndarray) else np.frombuffer(_as_bytes(corpus), np.uint8)
        self.counts += np.bincount(data, minlength=256).astype(np.uint64)
        self.total += int(data.size)


def compute_frequencies_gpu(data, device: int = 0) -> SymbolFrequencyTable:
    """compute_frequencies over a large byte blob on the GPU (fpg_byte_histogram)."""
    arr = data if isinstance(data, np.ndarray) else np.frombuffer(_as_bytes(data), np.uint8)
    counts = np.zeros(256, np.uint64)
    check(load_fpg().fpg_byte_histogram(ptr(arr), arr.size, device, ptr(counts)))
    t = SymbolFrequencyTable()
    t.counts = counts
    t.total = int(arr.size)
    return t


def compute_frequencies(words) -> SymbolFrequencyTable:
    """letter_model.hpp:33-45: counts over the concatenated words (or a blob)."""
    t = SymbolFrequencyTable()
    if isinstance(words, (bytes, str, np.ndarray)):
        t.add(words)
    else:
        for w in words:
            t.add(w)
    return t


class LetterSet:
    """letter_model.hpp:60-87: ordered symbols; slot q of c = index of c."""

    def __init__(self, symbols=b""):
        self._symbols = _as_bytes(symbols)
        self._slot = [-1] * 256
        for i, c in enumerate(self._symbols):
            if self._slot[c] != -1:
                raise ValueError("LetterSet: duplicate symbol in letter set")
            self._slot[c] = i

    def size(self) -> int:
        return len(self._symbols)

    def symbol(self, slot: int) -> int:
        return self._symbols[slot]

    def slot_of(self, c: int) -> int:
        return self._slot[c]

    def contains(self, c: int) -> bool:
        return self._slot[c] >= 0

    def symbols(self) -> bytes:
        return self._symbols


def select_letters(freq: SymbolFrequencyTable, count: int, strategy: LetterStrategy) -> LetterSet:
    """letter_model.hpp:94-134: rank by (count, byte) ascending; common = top."""
    ranked = sorted((int(freq.counts[c]), c) for c in range(256) if freq.counts[c])
    ranked = [c for _, c in ranked]
    if len(ranked) < count:
        raise ValueError(f"select_letters: collection has {len(ranked)} distinct symbols, need {count}")
    if strategy == LetterStrategy.Common:
        picked = [ranked[-1 - i] for i in range(count)]
    elif strategy == LetterStrategy.Rare:
        picked = ranked[:count]
    else:
        picked = [ranked[-1 - i] for i in range((count + 1) // 2)] + ranked[: count // 2]
    return LetterSet(bytes(picked))


def english_default_letters() -> str:
    """letter_model.hpp:137-139."""
    return "etaoinshrdlcumwfgypbvkjxqz"


# Standard English unigram frequencies (percent), a..z.
_EN_PCT = (8.167, 1.492, 2.782, 4.253, 12.702, 2.228, 2.015, 6.094, 6.966, 0.153, 0.772, 4.025, 2.406,
           6.749, 7.507, 1.929, 0.095, 5.987, 6.327, 9.056, 2.758, 0.978, 2.360, 0.150, 1.974, 0.074)


def english_letter_frequencies() -> list[tuple[int, float]]:
    """letter_model.hpp:147-157: (symbol, weight) pairs of English letters."""
    return [(ord("a") + i, w) for i, w in enumerate(_EN_PCT)]


# ---------------------------------------------------------------- schemes

def _letter_capacity(v: int, width: int, b: int, p: int) -> int:
    """Letters a scheme holds (fingerprint.hpp:84-100 with 16 -> W), -1 if
    the parameters are invalid."""
    if width not in (16, 32, 64):
        return -1
    if v == Variant.Occurrence:
        return width
    if v == Variant.OccurrenceHalved:
        return width // 2
    if v == Variant.Count:
        return -1 if b <= 0 or width % b else width // b
    if v == Variant.Position:
        if p <= 0 or p > width:
            return -1
        slots = width // p
        return slots + (width - slots * p)
    return -1


class Scheme:
    """fingerprint.hpp:57-162 with the width W as a parameter."""

    def __init__(self, variant: Variant, letters: LetterSet, b: int = 0, p: int = 0, width: int = 16):
        self._variant = Variant(variant)
        self._letters = letters if isinstance(letters, LetterSet) else LetterSet(letters)
        self._b, self._p, self._w = int(b), int(p), int(width)
        needed = Scheme.letter_capacity(self._variant, b or 2, p or 3, width)
        if self._letters.size() != needed:
            raise ValueError(f"scheme requires {needed} letters, got {self._letters.size()}")

    @staticmethod
    def occurrence(letters, width: int = 16) -> "Scheme":
        return Scheme(Variant.Occurrence, letters, 0, 0, width)

    @staticmethod
    def occurrence_halved(letters, width: int = 16) -> "Scheme":
        return Scheme(Variant.OccurrenceHalved, letters, 0, 0, width)

    @staticmethod
    def count(letters, bits_per_count: int = 2, width: int = 16) -> "Scheme":
        return Scheme(Variant.Count, letters, bits_per_count, 0, width)

    @staticmethod
    def position(letters, bits_per_position: int = 3, width: int = 16) -> "Scheme":
        return Scheme(Variant.Position, letters, 0, bits_per_position, width)

    @staticmethod
    def make(v: Variant, letters, bits_per_count: int = 2, bits_per_position: int = 3,
             width: int = 16) -> "Scheme":
        v = Variant(v)
        if v == Variant.Occurrence:
            return Scheme.occurrence(letters, width)
        if v == Variant.OccurrenceHalved:
            return Scheme.occurrence_halved(letters, width)
        if v == Variant.Count:
            return Scheme.count(letters, bits_per_count, width)
        return Scheme.position(letters, bits_per_position, width)

    @staticmethod
    def letter_capacity(v: Variant, b: int = 2, p: int = 3, width: int = 16) -> int:
        """fingerprint.hpp:84-100, 16 -> W.  Host arithmetic (the same rule as
        fpg_letter_capacity in libfpg.so; tests/test_host.py checks they
        agree), so building a Scheme never loads the CUDA library."""
        c = _letter_capacity(int(v), int(width), int(b), int(p))
        if c < 0:
            if Variant(v) == Variant.Count:
                raise ValueError(f"count scheme: bits per count must divide {width}")
            if Variant(v) == Variant.Position:
                raise ValueError(f"position scheme: bits per position must be in [1,{width}]")
            raise ValueError(f"invalid width {width}")
        return c

    def variant(self) -> Variant:
        return self._variant

    def letters(self) -> LetterSet:
        return self._letters

    def bits_per_count(self) -> int:
        return self._b

    def bits_per_position(self) -> int:
        return self._p

    def width(self) -> int:
        return self._w

    def position_slots(self) -> int:
        return self._w // self._p

    def extra_occurrence_slots(self) -> int:
        return self._w - self.position_slots() * self._p

    def supports(self, m: Metric) -> bool:
        return variant_supports(self._variant, m)

    def field_count(self) -> int:
        v = self._variant
        if v == Variant.Occurrence:
            return self._w
        if v == Variant.OccurrenceHalved:
            return self._w // 2
        if v == Variant.Count:
            return self._w // self._b
        return self.position_slots() + self.extra_occurrence_slots()

    def field_width(self, i: int) -> int:
        v = self._variant
        if v == Variant.Occurrence:
            return 1
        if v == Variant.OccurrenceHalved:
            return 2
        if v == Variant.Count:
            return self._b
        return self._p if i < self.position_slots() else 1

    def field_shift(self, i: int) -> int:
        if self._variant == Variant.Position:
            slots = self.position_slots()
            if i < slots:
                return self._w - self._p * (i + 1)
            return self.extra_occurrence_slots() - 1 - (i - slots)
        return self._w - self.field_width(0) * (i + 1)

    def c_struct(self) -> FpgScheme:
        s = FpgScheme()
        s.variant, s.width = int(self._variant), self._w
        s.bits_per_count, s.bits_per_position = self._b, self._p
        syms = self._letters.symbols()
        s.nletters = len(syms)
        for i, c in enumerate(syms):
            s.letters[i] = c
        return s


@dataclass(frozen=True)
class Fingerprint:
    """fingerprint.hpp:41-44 (bits zero-extended to 64)."""
    bits: int = 0


def render(f, scheme: Scheme) -> str:
    """fingerprint.hpp:305-317: slot-0 field leftmost, fields space-separated
    except for occurrence.  Pure formatting of bits the GPU produced."""
    bits = f.bits if isinstance(f, Fingerprint) else int(f)
    out = []
    for i in range(scheme.field_count()):
        if i and scheme.variant() != Variant.Occurrence:
            out.append(" ")
        w, sh = scheme.field_width(i), scheme.field_shift(i)
        out.extend("1" if (bits >> (sh + w - 1 - b)) & 1 else "0" for b in range(w))
    return "".join(out)


def build_many(words, scheme: Scheme, device: int = 0) -> np.ndarray:
    """build() (fingerprint.hpp:276-284) for every string, on the GPU (K1)."""
    blob, offsets = words if isinstance(words, tuple) else pack_strings(words)
    n = len(offsets) - 1
    out = np.zeros(max(n, 1), dtype=np.uint64)
    sch = scheme.c_struct()
    check(load_fpg().fpg_build_fingerprints(ptr(blob), ptr(offsets), n, ctypes.byref(sch), device,
                                            ptr(out)))
    return out[:n]


def build(s, scheme: Scheme, device: int = 0) -> Fingerprint:
    return Fingerprint(int(build_many([s], scheme, device)[0]))


# ---------------------------------------------------------------- queries

@dataclass
class QueryOptions:
    """dictionary.hpp:36-44 (positional order kept)."""
    metric: Metric = Metric.Hamming
    k: int = 1
    use_filter: bool = True
    length_prefilter: bool = False
    exhaustive: bool = False  # B200: byte-verify every pair, no pruning (naive-path timing)

    def c_struct(self, want_stats: bool) -> FpgQueryOptions:
        o = FpgQueryOptions()
        o.metric, o.k = int(self.metric), int(self.k)
        o.use_filter, o.length_prefilter = int(bool(self.use_filter)), int(bool(self.length_prefilter))
        o.want_stats = int(bool(want_stats))
        o.exhaustive = int(bool(self.exhaustive))
        return o


@dataclass
class QueryStats:
    """dictionary.hpp:19-34; accumulated with += like query_into (:116-117)."""
    compared: int = 0
    rejected_by_length: int = 0
    rejected_by_fingerprint: int = 0
    verified: int = 0
    matches: int = 0

    def __iadd__(self, o: "QueryStats") -> "QueryStats":
        self.compared += o.compared
        self.rejected_by_length += o.rejected_by_length
        self.rejected_by_fingerprint += o.rejected_by_fingerprint
        self.verified += o.verified
        self.matches += o.matches
        return self

    @staticmethod
    def from_row(row) -> "QueryStats":
        return QueryStats(*(int(x) for x in row))


@dataclass
class MatchCSR:
    """Batch result: matches of query i are word_ids[offsets[i]:offsets[i+1]],
    ascending input-order ids (dictionary.hpp:86,112)."""
    offsets: np.ndarray
    word_ids: np.ndarray

    def row(self, i: int) -> np.ndarray:
        return self.word_ids[int(self.offsets[i]):int(self.offsets[i + 1])]

    def __len__(self) -> int:
        return len(self.offsets) - 1


class _ResultOwner:
    """Owns a library-allocated fpg_result; frees it when the last numpy view
    of its arrays goes away (fpg_result_free)."""

    def __init__(self, res: FpgResult):
        self.res = res

    def __del__(self):
        try:
            load_fpg().fpg_result_free(ctypes.byref(self.res))
        except Exception:  # interpreter shutdown
            pass


def _take_result(res: FpgResult, want_stats: bool):
    """Wraps the library-owned CSR (and stats) as numpy arrays without a copy;
    the result is freed once all of them are released."""
    nq, total = int(res.nq), int(res.total)
    owner = _ResultOwner(res)

    def view(p, n, ctype, dtype):
        addr = ctypes.cast(p, ctypes.c_void_p).value
        if not n or not addr:
            return np.empty(n, dtype=dtype)
        buf = (ctype * n).from_address(addr)
        buf._owner = owner  # keeps the allocation alive as long as the view
        return np.frombuffer(buf, dtype=dtype)

    offsets = view(res.offsets, nq + 1, ctypes.c_uint64, np.uint64)
    ids = view(res.word_ids, total, ctypes.c_uint32, np.uint32)
    stats = view(res.stats, nq * 5, ctypes.c_uint64, np.uint64).reshape(nq, 5) if want_stats else None
    return MatchCSR(offsets, ids), stats


class GpuFingerprintedDictionary:
    """FingerprintedDictionary (dictionary.hpp:47-125) on B200s.

    ``words`` is a sequence of str/bytes or a pre-packed (blob, offsets)
    pair.  ``devices`` shards the collection into contiguous input-order id
    ranges, one per entry.  Immutable after construction; ``query*`` may be
    called from several threads.
    """

    def __init__(self, words, scheme: Scheme, devices: Sequence[int] = (0,), id_base: int = 0,
                 keep_words: bool = True):
        self._lib = load_fpg()
        self._scheme = scheme
        blob, offsets = words if isinstance(words, tuple) else pack_strings(words)
        self._blob, self._offsets = (blob, offsets) if keep_words else (None, None)
        self._n = len(offsets) - 1
        devs = (ctypes.c_int32 * len(devices))(*devices)
        sch = scheme.c_struct()
        h = ctypes.c_void_p()
        check(self._lib.fpg_dict_create(ptr(blob), ptr(offsets), self._n, ctypes.byref(sch), devs,
                                        len(devices), id_base, ctypes.byref(h)))
        self._h = h
        self._batch = None
        self._batches = weakref.WeakSet()  # live Batch objects: closed before the dictionary

    @classmethod
    def from_text(cls, text, scheme: Scheme, devices: Sequence[int] = (0,), id_base: int = 0):
        """The dictionary of a newline-separated word text (read_word_lines,
        corpus.hpp:116-125), split into words on the GPU(s).  ``text`` is
        bytes, a uint8 array or a path; words() is not kept."""
        if isinstance(text, (str,)) or hasattr(text, "__fspath__"):
            with open(text, "rb") as f:
                text = f.read()
        data = text if isinstance(text, np.ndarray) else np.frombuffer(bytes(text), np.uint8)
        self = cls.__new__(cls)
        self._lib = load_fpg()
        self._scheme = scheme
        self._blob = self._offsets = None
        devs = (ctypes.c_int32 * len(devices))(*devices)
        sch = scheme.c_struct()
        h = ctypes.c_void_p()
        check(self._lib.fpg_dict_create_from_text(ptr(data), data.size, ctypes.byref(sch), devs, len(devices),
                                                  id_base, ctypes.byref(h)))
        self._h = h
        self._batch = None
        self._batches = weakref.WeakSet()
        n = ctypes.c_uint64()
        check(self._lib.fpg_dict_size(h, ctypes.byref(n)))
        self._n = n.value
        return self

    def close(self) -> None:
        if getattr(self, "_batch", None):
            self._lib.fpg_batch_destroy(self._batch)
            self._batch = None
        for b in list(getattr(self, "_batches", ())):  # the C ABI refuses to drop a dict with live batches
            b.close()
        if getattr(self, "_h", None):
            self._lib.fpg_dict_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # accessors (dictionary.hpp:58-62)
    def size(self) -> int:
        return self._n

    def scheme(self) -> Scheme:
        return self._scheme

    def words(self) -> list[bytes]:
        if self._blob is None:
            raise ValueError("dictionary built with keep_words=False")
        o = self._offsets
        return [bytes(self._blob[int(o[i]):int(o[i + 1])]) for i in range(self._n)]

    def prints_array(self) -> np.ndarray:
        out = np.zeros(max(self._n, 1), dtype=np.uint64)
        check(self._lib.fpg_dict_prints(self._h, ptr(out)))
        return out[: self._n]

    def prints(self) -> list[Fingerprint]:
        return [Fingerprint(int(x)) for x in self.prints_array()]

    def scan_shape(self) -> dict:
        """K2 path of this dictionary: bit-sliced or generic, and the sig' field count."""
        sl, sg = ctypes.c_int32(), ctypes.c_int32()
        check(self._lib.fpg_dict_scan_shape(self._h, ctypes.byref(sl), ctypes.byref(sg)))
        return {"sliced": bool(sl.value), "sig_fields": sg.value}

    def build_seconds(self) -> float:
        s = ctypes.c_double()
        check(self._lib.fpg_dict_build_seconds(self._h, ctypes.byref(s)))
        return s.value

    def build_profile(self, shard: int = 0) -> list[dict]:
        """Construction stages of one shard: name, device ms (CUDA events)
        and algorithmic HBM bytes (fpg_dict_build_profile)."""
        from ._lib import FpgBuildStage

        arr = (FpgBuildStage * 8)()
        n = ctypes.c_int32()
        check(self._lib.fpg_dict_build_profile(self._h, shard, arr, 8, ctypes.byref(n)))
        return [{"name": arr[i].name.decode(), "ms": arr[i].ms, "bytes": arr[i].bytes} for i in range(min(n.value, 8))]

    # queries
    def query_batch(self, queries, opt: QueryOptions, per_query_stats: bool = False):
        """All queries in one GPU pass.  Returns (MatchCSR, stats[nq,5] | None)."""
        qblob, qoffs = queries if isinstance(queries, tuple) else pack_strings(queries)
        nq = len(qoffs) - 1
        o = opt.c_struct(per_query_stats)
        res = FpgResult()
        check(self._lib.fpg_query_batch(self._h, ptr(qblob), ptr(qoffs), nq, ctypes.byref(o),
                                        ctypes.byref(res)))
        return _take_result(res, per_query_stats)

    def query_into(self, pattern, opt: QueryOptions, matches: list, stats: QueryStats | None = None):
        """dictionary.hpp:75-118: clears and refills `matches`; accumulates stats."""
        matches.clear()
        csr, st = self.query_batch([pattern], opt, per_query_stats=stats is not None)
        matches.extend(int(x) for x in csr.row(0))
        if stats is not None:
            stats += QueryStats.from_row(st[0])

    def query(self, pattern, opt: QueryOptions = None, stats: QueryStats | None = None) -> list[int]:
        """dictionary.hpp:66-71."""
        m: list[int] = []
        self.query_into(pattern, opt or QueryOptions(), m, stats)
        return m

    # staged API (device-resident measurement)
    def batch(self) -> "Batch":
        b = Batch(self)
        self._batches.add(b)
        return b


def csr_merge_device(device: int, parts, nq: int, out_offsets: int, out_ids: int, stream: int = 0) -> None:
    """fpg_csr_merge_device: parts = [(offsets_ptr, ids_ptr), ...] of per-shard
    CSRs in `device` memory (shard order), merged into the device buffers
    out_offsets (nq + 1 uint64) and out_ids, asynchronously on `stream`."""
    n = len(parts)
    offs = (ctypes.c_void_p * n)(*[ctypes.c_void_p(o) for o, _ in parts])
    ids = (ctypes.c_void_p * n)(*[ctypes.c_void_p(i) for _, i in parts])
    check(load_fpg().fpg_csr_merge_device(device, n, offs, ids, nq, ctypes.c_void_p(out_offsets),
                                          ctypes.c_void_p(out_ids), ctypes.c_void_p(stream)))


class Batch:
    """fpg_batch_*: upload (H2D) / run (device only) / download (D2H)."""

    def __init__(self, d: GpuFingerprintedDictionary):
        self._lib = d._lib
        self._d = d
        h = ctypes.c_void_p()
        check(self._lib.fpg_batch_create(d._h, ctypes.byref(h)))
        self._h = h

    def upload(self, qblob: np.ndarray, qoffs: np.ndarray) -> None:
        self._qblob, self._qoffs = qblob, qoffs  # keep alive
        check(self._lib.fpg_batch_upload(self._h, ptr(qblob), ptr(qoffs), len(qoffs) - 1))

    def run(self, opt: QueryOptions, want_stats: bool = False) -> None:
        self._want_stats = want_stats
        o = opt.c_struct(want_stats)
        check(self._lib.fpg_batch_run(self._h, ctypes.byref(o)))

    def download(self):
        res = FpgResult()
        check(self._lib.fpg_batch_download(self._h, ctypes.byref(res)))
        return _take_result(res, getattr(self, "_want_stats", False))

    def timing(self, shard: int = 0) -> dict:
        run_ms, filt_ms = ctypes.c_double(), ctypes.c_double()
        ex, sv, ln = ctypes.c_uint64(), ctypes.c_uint64(), ctypes.c_uint64()
        check(self._lib.fpg_batch_last_timing(self._h, shard, ctypes.byref(run_ms), ctypes.byref(filt_ms),
                                              ctypes.byref(ex), ctypes.byref(sv), ctypes.byref(ln)))
        cand, scan = ctypes.c_uint64(), ctypes.c_uint64()
        check(self._lib.fpg_batch_last_candidates(self._h, shard, ctypes.byref(cand)))
        check(self._lib.fpg_batch_last_scanned(self._h, shard, ctypes.byref(scan)))
        scan_x = ctypes.c_uint64()
        check(self._lib.fpg_batch_last_scanned_exact(self._h, shard, ctypes.byref(scan_x)))
        ver_ms, recs, rounds, plan_ms = ctypes.c_double(), ctypes.c_uint64(), ctypes.c_uint32(), ctypes.c_double()
        check(self._lib.fpg_batch_last_verify(self._h, shard, ctypes.byref(ver_ms), ctypes.byref(recs),
                                              ctypes.byref(rounds), ctypes.byref(plan_ms)))
        return {"run_ms": run_ms.value, "filter_ms": filt_ms.value, "executed_pairs": ex.value,
                "survivors": sv.value, "launches": ln.value, "candidates": cand.value, "scanned_pairs": scan.value,
                "scanned_pairs_exact": scan_x.value, "verify_ms": ver_ms.value, "candidate_records": recs.value,
                "verify_rounds": rounds.value, "plan_ms": plan_ms.value}

    def host_ms(self) -> dict:
        """Host-side ms of the last upload, download (D2H wait) and result
        assembly (the host gather of shard rows)."""
        u, d, a = ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
        check(self._lib.fpg_batch_last_host_ms(self._h, ctypes.byref(u), ctypes.byref(d), ctypes.byref(a)))
        return {"upload_ms": u.value, "download_ms": d.value, "assemble_ms": a.value}

    def device_csr(self, shard: int = 0) -> dict:
        """Device pointers of the last run's CSR on `shard` (global ids):
        {device, nq, total, offsets, ids}; valid until the next run."""
        dev, total = ctypes.c_int32(), ctypes.c_uint64()
        off, ids = ctypes.c_void_p(), ctypes.c_void_p()
        check(self._lib.fpg_batch_device_csr(self._h, shard, ctypes.byref(dev), ctypes.byref(total),
                                             ctypes.byref(off), ctypes.byref(ids)))
        return {"device": dev.value, "nq": len(self._qoffs) - 1, "total": total.value,
                "offsets": off.value or 0, "ids": ids.value or 0}

    def close(self) -> None:
        if getattr(self, "_h", None):
            self._lib.fpg_batch_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
