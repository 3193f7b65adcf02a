"""GPU parity: libfpg.so (through the C ABI) vs the CPU oracle on the same
seeded inputs.  Bit-exact for fingerprints, match sets and QueryStats."""
import json
from pathlib import Path

import numpy as np
import pytest

from oracle.oracle import oscheme, pack
from paper_1711_08475_b200 import (GpuFingerprintedDictionary, LetterSet, Metric, QueryOptions,
                                   QueryStats, Scheme, Variant, build, build_many, render, variant_supports)
from paper_1711_08475_b200.corpus import (CELLS, generate_dictionary, generate_queries, make_scheme,
                                          subsample)

pytestmark = pytest.mark.gpu
GOLD = json.loads((Path(__file__).parent / "golden" / "reference_vectors.json").read_text())


def osch(s: Scheme):
    return oscheme(int(s.variant()), s.letters().symbols(), s.width(), s.bits_per_count() or 2,
                   s.bits_per_position() or 3)


def fixture_scheme(rec, width=16):
    return Scheme.make(Variant(rec["variant"]), LetterSet(rec["letters"]), rec["b"], rec["p"], width)


def assert_same(csr, st, ref_off, ref_ids, ref_st=None):
    assert np.array_equal(csr.offsets, ref_off), "per-query match counts differ"
    assert np.array_equal(csr.word_ids, ref_ids), "match ids differ"
    if ref_st is not None:
        assert np.array_equal(st, ref_st), "QueryStats differ"


# ---------------------------------------------------------------- K1 vs the reference fixtures

def test_golden_instance_renders():
    # fingerprint_test.cpp:60-66 / acceptance_test.cpp:97-113
    want = ["1110111000010000", "01 10 01 00 10 11 10 00", "01 01 01 00 01 10 01 00", "111 011 100 111 000 1"]
    for rec, w in zip(GOLD["schemes"][:4], want):
        s = fixture_scheme(rec)
        assert render(build("instance", s), s) == w


def test_golden_tiny_strings():
    occ, halved, count, pos = (fixture_scheme(r) for r in GOLD["schemes"][:4])
    assert build("", occ).bits == 0 and build("", halved).bits == 0 and build("", count).bits == 0
    assert render(build("", pos), pos) == "111 111 111 111 111 0"          # fingerprint_test.cpp:73
    assert render(build("e", halved), halved) == "01 00 00 00 00 00 00 00"  # :75-76
    assert render(build("e" + "z" * 19, pos), pos) == "000 111 111 111 111 0"  # :83
    assert render(build("zzzzzze", pos), pos) == "110 111 111 111 111 0"    # :88
    assert build("zzzzzzze", pos) == build("zzzzzzzz", pos)                 # :85-87
    assert render(build("eeee", count), count) == "11 00 00 00 00 00 00 00"  # :94-96
    assert render(build("ee", count), count) == "10 00 00 00 00 00 00 00"


@pytest.mark.parametrize("idx", range(len(GOLD["schemes"])))
def test_prints_match_reference(idx):
    rec = GOLD["schemes"][idx]
    words = [bytes.fromhex(h) for h in GOLD["words"]]
    s = fixture_scheme(rec)
    got = build_many(words, s)
    assert [int(x) for x in got] == rec["prints"]
    # and through the dictionary (bucketed layout, input-order prints())
    with GpuFingerprintedDictionary(words, s) as d:
        assert [int(x) for x in d.prints_array()] == rec["prints"]


@pytest.mark.parametrize("variant,width,b,p", [
    (Variant.Occurrence, 32, 2, 3), (Variant.Occurrence, 64, 2, 3),
    (Variant.OccurrenceHalved, 32, 2, 3), (Variant.OccurrenceHalved, 64, 2, 3),
    (Variant.Count, 32, 2, 3), (Variant.Count, 64, 4, 3), (Variant.Count, 64, 2, 3),
    (Variant.Position, 32, 2, 3), (Variant.Position, 64, 2, 3), (Variant.Position, 64, 2, 5),
])
def test_prints_wide_vs_oracle(oracle, variant, width, b, p):
    rng = np.random.default_rng(width * 10 + int(variant))
    alphabet = bytes(range(33, 33 + 70))
    cap = Scheme.letter_capacity(variant, b, p, width)
    letters = bytes(rng.permutation(np.frombuffer(alphabet, np.uint8))[:cap])
    s = Scheme.make(variant, LetterSet(letters), b, p, width)
    words = [bytes(rng.choice(np.frombuffer(alphabet, np.uint8), rng.integers(0, 120))) for _ in range(3000)]
    blob, offs = pack(words)
    assert np.array_equal(build_many((blob, offs), s), oracle.build_many(blob, offs, osch(s)))


# ---------------------------------------------------------------- K2/K3 vs reference fixtures

def _fixture_case(q):
    rec = next(r for r in GOLD["schemes"] if r["name"] == q["scheme"])
    return rec


@pytest.mark.parametrize("case", range(len(GOLD["queries"])))
def test_queries_match_reference_fixture(case, exact_path):
    q = GOLD["queries"][case]
    s = fixture_scheme(_fixture_case(q))
    words = [bytes.fromhex(h) for h in GOLD["query_dict"]]
    pats = [bytes.fromhex(h) for h in GOLD["query_patterns"]]
    opt = QueryOptions(Metric(q["metric"]), q["k"], q["use_filter"], q["length_prefilter"])
    with GpuFingerprintedDictionary(words, s) as d:
        csr, st = d.query_batch(pats, opt, per_query_stats=True)
    assert_same(csr, st, np.array(q["offsets"], np.uint64), np.array(q["ids"], np.uint32),
                np.array(q["stats"], np.uint64))


def test_query_api_semantics():
    """dictionary_test.cpp:64-84, :110-139, :160-170 through the mirror API."""
    occ = Scheme.occurrence(LetterSet("etaoinshrdlcumwf"))
    with GpuFingerprintedDictionary(["run"], occ) as d:
        st = QueryStats()
        assert d.query("ran", QueryOptions(Metric.Hamming, 1), st) == [0]
        assert st.rejected_by_fingerprint == 0 and st.verified == 1
        st0 = QueryStats()
        assert d.query("ran", QueryOptions(Metric.Hamming, 0), st0) == []
        assert st0.compared == st0.rejected_by_length + st0.rejected_by_fingerprint + st0.verified
        m = [99]
        d.query_into("run", QueryOptions(), m)
        assert m == [0]
    pos = Scheme.position(LetterSet("abcdef"), 3)
    with GpuFingerprintedDictionary(["abcdef", "ghijkl"], pos) as d:
        with pytest.raises(ValueError):
            d.query("abcdef", QueryOptions(Metric.Levenshtein, 1, True, False))
        assert d.query("abcdef", QueryOptions(Metric.Levenshtein, 1, False, False)) == [0]
    with GpuFingerprintedDictionary([], occ) as d:
        st = QueryStats()
        assert d.query("ran", QueryOptions(), st) == [] and st.compared == 0


# ---------------------------------------------------------------- configs vs the oracle

def _cfg_inputs(cfg, n, nq):
    blob, offs = generate_dictionary(cfg, n=n)
    qblob, qoffs = generate_queries(cfg, blob, offs, nq=nq)
    return blob, offs, qblob, qoffs


@pytest.mark.parametrize("cfg,n,nq", [(1, 100_000, 1000), (2, 200_000, 600), (3, 200_000, 600), (4, 50_000, 300),
                                      (5, 200_000, 600)])
def test_config_cells_vs_oracle(oracle, cfg, n, nq, exact_path):
    blob, offs, qblob, qoffs = _cfg_inputs(cfg, n, nq)
    for variant, width, b, p, metric in CELLS[cfg]:
        s = make_scheme(blob, variant, width, b, p)
        with GpuFingerprintedDictionary((blob, offs), s) as d:
            assert np.array_equal(d.prints_array(), oracle.build_many(blob, offs, osch(s)))
            for pre in ((True, False) if metric == Metric.Levenshtein else (False,)):
                opt = QueryOptions(metric, 1, True, pre)
                csr, st = d.query_batch((qblob, qoffs), opt, per_query_stats=True)
                o_off, o_ids, o_st = oracle.query_batch(blob, offs, qblob, qoffs, osch(s), metric, 1, True, pre)
                assert_same(csr, st, o_off, o_ids, o_st)


@pytest.mark.parametrize("metric", [Metric.Hamming, Metric.Levenshtein])
@pytest.mark.parametrize("k", [0, 1, 2, 3])
def test_filter_off_and_k0(oracle, metric, k, exact_path):
    """k = 0..3 (k >= 2 runs the generic kernel and the banded verifier), filter on/off."""
    blob, offs, qblob, qoffs = _cfg_inputs(2, 50_000, 300)
    s = make_scheme(blob, Variant.Count, 16)
    with GpuFingerprintedDictionary((blob, offs), s) as d:
        for use_filter in (True, False):
            opt = QueryOptions(metric, k, use_filter, True)
            csr, st = d.query_batch((qblob, qoffs), opt, per_query_stats=True)
            o = oracle.query_batch(blob, offs, qblob, qoffs, osch(s), metric, k, use_filter, True)
            assert_same(csr, st, *o)
    naive_off, naive_ids = oracle.naive_scan_batch(blob, offs, qblob, qoffs, metric, k)
    assert np.array_equal(csr.offsets, naive_off) and np.array_equal(csr.word_ids, naive_ids)


def test_edge_strings(oracle, exact_path):
    """Empty strings, 1-byte strings, zero bytes, 0xff, duplicates, long strings."""
    rng = np.random.default_rng(7)
    words = [b"", b"", b"a", b"\x00", b"a\x00", b"\x00a", b"\xff" * 3, b"ab", b"ba"]
    words += [bytes(rng.integers(0, 4, rng.integers(0, 40)).astype(np.uint8)) for _ in range(3000)]
    words += [bytes(rng.integers(97, 100, 4096).astype(np.uint8)), bytes(rng.integers(97, 100, 4095).astype(np.uint8))]
    words += words[:50]  # duplicates keep distinct ids
    pats = [b"", b"a", b"\x00", b"\x00\x00", words[-3], words[-53][:-1] + b"\x07"]
    pats += [bytes(rng.integers(0, 4, rng.integers(0, 40)).astype(np.uint8)) for _ in range(300)]
    blob, offs = pack(words)
    qblob, qoffs = pack(pats)
    s = Scheme.occurrence(LetterSet(bytes([0, 1, 2, 3, 97, 98, 99, 255] + list(range(10, 18)))))
    with GpuFingerprintedDictionary((blob, offs), s) as d:
        for metric in (Metric.Hamming, Metric.Levenshtein):
            for pre in (True, False):
                opt = QueryOptions(metric, 1, True, pre)
                csr, st = d.query_batch((qblob, qoffs), opt, per_query_stats=True)
                assert_same(csr, st, *oracle.query_batch(blob, offs, qblob, qoffs, osch(s), metric, 1, True, pre))


@pytest.mark.parametrize("variant,width", [(Variant.Occurrence, 16), (Variant.Count, 32), (Variant.Position, 64)])
def test_k_above_one_other_schemes(oracle, variant, width):
    """k = 2 on bit-sliced dictionaries of other widths, Hamming and (where the
    scheme filters it) Levenshtein, without and with the length prefilter."""
    blob, offs, qblob, qoffs = _cfg_inputs(5, 40_000, 200)
    s = make_scheme(blob, variant, width)
    with GpuFingerprintedDictionary((blob, offs), s) as d:
        for metric in (Metric.Hamming, Metric.Levenshtein):
            use_filter = variant_supports(variant, metric)
            for pre in (True, False):
                csr, st = d.query_batch((qblob, qoffs), QueryOptions(metric, 2, use_filter, pre), per_query_stats=True)
                assert_same(csr, st, *oracle.query_batch(blob, offs, qblob, qoffs, osch(s), metric, 2, use_filter, pre))


def test_concurrent_query_batches(oracle):
    """Concurrent const queries are safe in the reference (README.md:124-125):
    four host threads share one dictionary handle, each with its own batch."""
    import threading

    blob, offs, qblob, qoffs = _cfg_inputs(2, 80_000, 300)
    s = make_scheme(blob, Variant.Count, 16)
    want = oracle.query_batch(blob, offs, qblob, qoffs, osch(s), Metric.Levenshtein, 1, True, True)
    errors = []
    with GpuFingerprintedDictionary((blob, offs), s) as d:
        def worker():
            try:
                for _ in range(5):
                    csr, st = d.query_batch((qblob, qoffs), QueryOptions(Metric.Levenshtein, 1, True, True), True)
                    assert_same(csr, st, *want)
            except Exception as e:  # reported below
                errors.append(e)
        th = [threading.Thread(target=worker) for _ in range(4)]
        for t in th:
            t.start()
        for t in th:
            t.join()
    assert not errors, errors[0]


def test_too_long_and_invalid_args():
    s = Scheme.occurrence(LetterSet("etaoinshrdlcumwf"))
    with pytest.raises(ValueError):
        GpuFingerprintedDictionary([b"a" * 4097], s)
    with pytest.raises(ValueError):
        Scheme.occurrence(LetterSet("abc"))
    with pytest.raises(ValueError):
        Scheme.count(LetterSet("etaoinsh"), 3)
    with GpuFingerprintedDictionary(["abc"], s) as d:
        assert d.query("abd", QueryOptions(Metric.Hamming, 2)) == [0]  # k >= 2: generic kernel
        with pytest.raises(Exception):
            d.query("abc", QueryOptions(Metric.Hamming, 9))  # k > kMaxK is not built for the GPU
        with pytest.raises(ValueError):
            d.query("abc", QueryOptions(Metric.Hamming, -1))
        csr, st = d.query_batch([], QueryOptions(), per_query_stats=True)
        assert len(csr) == 0 and st.shape == (0, 5)


def test_shards_equal_single_device(oracle, exact_path):
    """Dictionary sharded over [0,0,0] (three shards on one GPU, independent
    kernels) gives the single-shard answer with rebased ids."""
    blob, offs, qblob, qoffs = _cfg_inputs(5, 100_000, 400)
    s = make_scheme(blob, Variant.Occurrence, 16)
    opt = QueryOptions(Metric.Levenshtein, 1, True, False)
    with GpuFingerprintedDictionary((blob, offs), s, devices=(0,)) as d1, \
         GpuFingerprintedDictionary((blob, offs), s, devices=(0, 0, 0)) as d3:
        a = d1.query_batch((qblob, qoffs), opt, per_query_stats=True)
        b = d3.query_batch((qblob, qoffs), opt, per_query_stats=True)
        assert np.array_equal(d1.prints_array(), d3.prints_array())
    assert np.array_equal(a[0].offsets, b[0].offsets) and np.array_equal(a[0].word_ids, b[0].word_ids)
    assert np.array_equal(a[1], b[1])


def test_output_regrowth_many_matches(oracle):
    """Config-3 short queries match tens of thousands of words each; the
    result buffer starts at 2^20 pairs and must regrow and rescan."""
    blob, offs = generate_dictionary(3, n=400_000)
    words = [b"e", b"t", b"ea", b"te", b"th", b"an", b"a"] * 40
    qblob, qoffs = pack(words)
    s = make_scheme(blob, Variant.Occurrence, 16)
    with GpuFingerprintedDictionary((blob, offs), s) as d:
        csr, st = d.query_batch((qblob, qoffs), QueryOptions(Metric.Levenshtein, 1, True, True), True)
    assert csr.offsets[-1] > (1 << 20)
    assert_same(csr, st, *oracle.query_batch(blob, offs, qblob, qoffs, osch(s), Metric.Levenshtein, 1, True, True))


@pytest.mark.parametrize("limit", [5000, 60_000])
def test_candidate_buffer_rounds(oracle, monkeypatch, limit):
    """K2 hands its candidates to K3 through a bounded record buffer.  With
    the buffer limited to a few thousand records (FPG_CAND_MAX) the run
    overflows, is redone with a grown buffer and then in several K2 + K3
    rounds; results and QueryStats must not change."""
    monkeypatch.setenv("FPG_CAND_MAX", str(limit))
    blob, offs = generate_dictionary(3, n=150_000)
    qb2, qo2 = generate_queries(3, blob, offs, nq=300)
    pats = [b"e", b"ea", b"th", b"and"]
    qblob, qoffs = pack(pats + [bytes(qb2[int(qo2[i]):int(qo2[i + 1])]) for i in range(300)])
    s = make_scheme(blob, Variant.Occurrence, 16)
    with GpuFingerprintedDictionary((blob, offs), s) as d:
        b = d.batch()
        b.upload(qblob, qoffs)
        for metric in (Metric.Hamming, Metric.Levenshtein):
            b.run(QueryOptions(metric, 1, True, True), want_stats=True)
            t = b.timing()
            csr, st = b.download()
            assert t["candidate_records"] <= limit
            if limit < 60_000:
                assert t["verify_rounds"] > 1
            assert_same(csr, st, *oracle.query_batch(blob, offs, qblob, qoffs, osch(s), metric, 1, True, True))
        b.close()


@pytest.mark.parametrize("no_barrier", ["0", "1"])
def test_tiles_with_and_without_barriers(oracle, monkeypatch, no_barrier):
    """K2 runs a tile's warps either between two CTA barriers or, for small
    batches, without barriers (double-buffered query data, the first warp out
    sets up the next tile).  Both variants forced on the same inputs,
    including tiles with fewer slab groups than warps and many tiles per CTA."""
    monkeypatch.setenv("FPG_NO_BARRIER", no_barrier)
    for cfg, n, nq in [(2, 120_000, 900), (3, 150_000, 700), (5, 300_000, 3000)]:
        blob, offs = generate_dictionary(cfg, n=n)
        qblob, qoffs = generate_queries(cfg, blob, offs, nq=nq)
        for variant, width, metric in [(Variant.Occurrence, 16, Metric.Hamming), (Variant.Count, 16, Metric.Levenshtein)]:
            s = make_scheme(blob, variant, width)
            with GpuFingerprintedDictionary((blob, offs), s) as d:
                csr, st = d.query_batch((qblob, qoffs), QueryOptions(metric, 1, True, True), True)
            assert_same(csr, st, *oracle.query_batch(blob, offs, qblob, qoffs, osch(s), metric, 1, True, True))


@pytest.mark.parametrize("hist", ["0", "1"])
def test_query_stats_from_histograms_or_counters(oracle, monkeypatch, hist):
    """QueryStats::verified of 16-bit schemes comes from per-length fingerprint
    histograms (k_fp_stats) or, with FPG_HIST_STATS=0, from K2's survivor
    counters (generic instantiation, no exact path); both must equal the
    oracle for every variant, metric, k in {0, 1} and prefilter setting."""
    monkeypatch.setenv("FPG_HIST_STATS", hist)
    blob, offs = generate_dictionary(5, n=200_000)
    qblob, qoffs = generate_queries(5, blob, offs, nq=1500)
    for variant in (Variant.Occurrence, Variant.OccurrenceHalved, Variant.Count, Variant.Position):
        s = make_scheme(blob, variant, 16)
        with GpuFingerprintedDictionary((blob, offs), s) as d:
            for metric in (Metric.Hamming, Metric.Levenshtein):
                if not variant_supports(variant, metric):
                    continue
                for k, pre in [(1, True), (0, True), (1, False)]:
                    csr, st = d.query_batch((qblob, qoffs), QueryOptions(metric, k, True, pre), True)
                    assert_same(csr, st, *oracle.query_batch(blob, offs, qblob, qoffs, osch(s), metric, k, True, pre))


def test_k4_segment_size_classes(oracle, exact_path):
    """K4 sorts each query's matches by word id in one of three ways: <= 32
    (warp bitonic), 33..4096 (one CTA, shared-memory bitonic) and larger
    (value-range buckets, per-warp sorts), with a CUB fallback when one bucket
    overflows.  The dictionary mixes duplicate runs so that one query hits
    each class, and its ids are placed so the last query's bucket overflows."""
    rng = np.random.default_rng(11)
    words = [bytes(rng.integers(97, 123, size=int(rng.integers(3, 9)), dtype=np.uint8)) for _ in range(60_000)]
    # 20 / 900 / 9000 copies at random (disjoint) ids past the first 3000
    at = rng.permutation(np.arange(3000, len(words) - 1))
    for w, (lo, hi) in [(b"qq", (0, 20)), (b"zx", (20, 920)), (b"kj", (920, 9920))]:
        for i in at[lo:hi]:
            words[int(i)] = w
    # skew: 3000 copies of "vw" packed at the front, one at the very end
    words[:3000] = [b"vw"] * 3000
    words[-1] = b"vw"
    blob, offs = pack(words)
    qblob, qoffs = pack([b"qq", b"zx", b"kj", b"vw", b"ab"])
    s = make_scheme(blob, Variant.Occurrence, 16)
    for metric in (Metric.Hamming, Metric.Levenshtein):
        with GpuFingerprintedDictionary((blob, offs), s) as d:
            csr, st = d.query_batch((qblob, qoffs), QueryOptions(metric, 1, True, True), True)
        counts = np.diff(csr.offsets)
        if metric == Metric.Hamming:  # one query per size class
            assert counts[0] <= 32 < counts[1] <= 4096 < counts[2] and counts[3] > 3000
        assert_same(csr, st, *oracle.query_batch(blob, offs, qblob, qoffs, osch(s), metric, 1, True, True))


def test_staged_batch_reruns_across_options(oracle, exact_path):
    """One upload, several runs (fpg_batch_run) with options whose outputs
    differ in size and shape: the cached tile plan and the K4 path choice
    (segmented vs radix sort, chosen per batch) must follow the options."""
    blob, offs = generate_dictionary(3, n=60_000)
    pats = [b"e", b"ea", b"th"] * 3
    qb2, qo2 = generate_queries(3, blob, offs, nq=200)
    qblob, qoffs = pack(pats + [bytes(qb2[int(qo2[i]):int(qo2[i + 1])]) for i in range(200)])
    s = make_scheme(blob, Variant.Occurrence, 16)
    with GpuFingerprintedDictionary((blob, offs), s) as d:
        b = d.batch()
        b.upload(qblob, qoffs)
        for metric, k, pre in [(Metric.Levenshtein, 1, True), (Metric.Hamming, 0, True),
                               (Metric.Levenshtein, 1, False), (Metric.Hamming, 1, True), (Metric.Levenshtein, 0, True)]:
            b.run(QueryOptions(metric, k, True, pre), want_stats=True)
            csr, st = b.download()
            assert_same(csr, st, *oracle.query_batch(blob, offs, qblob, qoffs, osch(s), metric, k, True, pre))
            # exhaustive (no pruning, every pair byte-verified): same matches, filter-off stats
            b.run(QueryOptions(metric, k, False, pre, exhaustive=True), want_stats=True)
            csr, st = b.download()
            assert_same(csr, st, *oracle.query_batch(blob, offs, qblob, qoffs, osch(s), metric, k, False, pre))


@pytest.mark.slow
def test_config2_full_dictionary_subsample(oracle):
    """Full config 2 (1e6 words, 10,000 queries) on the GPU; every 10th query
    checked against the oracle, and the batch is self-consistent:
    filter on == filter off, 1 shard == 2 shards."""
    blob, offs, qblob, qoffs = _cfg_inputs(2, None, None)
    s = make_scheme(blob, Variant.Count, 16)
    opt = QueryOptions(Metric.Levenshtein, 1, True, True)
    with GpuFingerprintedDictionary((blob, offs), s) as d:
        csr, st = d.query_batch((qblob, qoffs), opt, per_query_stats=True)
        off_nf, _ = d.query_batch((qblob, qoffs), QueryOptions(Metric.Levenshtein, 1, False, True))
    sb, so, idx = subsample(qblob, qoffs, 10)
    o_off, o_ids, o_st = oracle.query_batch(blob, offs, sb, so, osch(s), Metric.Levenshtein, 1, True, True)
    for j, q in enumerate(idx):
        assert np.array_equal(csr.row(q), o_ids[int(o_off[j]):int(o_off[j + 1])])
        assert np.array_equal(st[q], o_st[j])
    assert np.array_equal(csr.offsets, off_nf.offsets) and np.array_equal(csr.word_ids, off_nf.word_ids)
    with GpuFingerprintedDictionary((blob, offs), s, devices=(0, 0)) as d2:
        c2, _ = d2.query_batch((qblob, qoffs), opt)
    assert np.array_equal(csr.word_ids, c2.word_ids)


@pytest.mark.gpu
def test_cpp_drop_in_queries(tmp_path):
    """The C++ FingerprintedDictionary alias (b200.hpp) answers query /
    query_batch like a brute-force scan and throws invalid_argument for
    position + Levenshtein, as dictionary.hpp:78-79 does."""
    import subprocess

    from conftest import build_api_check

    exe = build_api_check(tmp_path)
    out = subprocess.run([str(exe), "gpu"], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr + out.stdout
    assert "api_check gpu: ok" in out.stdout


@pytest.mark.gpu
def test_cpp_reference_extension():
    """Reference caller code with the reference's FingerprintedDictionary,
    naive_scan and the GPU dictionary (b200_ref.hpp) in one translation
    unit: prints, matches and QueryStats equal for every variant x metric
    the reference filters, and every GPU match passes the reference's
    can_reject with the GPU dictionary's tables() (tests/cpp/api_check_ref.cpp,
    prebuilt by __graft_entry__.build() where the reference tree exists)."""
    import subprocess

    from conftest import API_CHECK_REF_BIN, REF_INCLUDE, build_api_check_ref

    exe = API_CHECK_REF_BIN
    if (REF_INCLUDE / "fingerprints" / "dictionary.hpp").exists():
        exe = build_api_check_ref()
    if not exe.exists():
        pytest.skip("api_check_ref was not prebuilt (no reference tree where build() ran)")
    out = subprocess.run([str(exe), "gpu"], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr + out.stdout
    assert "api_check_ref gpu: ok" in out.stdout


@pytest.mark.parametrize("text", [b"", b"\n", b"a", b"a\n", b"a\n\nbc\r\nd", b"\n\n\n", b"xy\nz"])
def test_dictionary_from_text_edges(text):
    """fpg_dict_create_from_text splits like read_word_lines (corpus.hpp:116-125)."""
    words = text.split(b"\n")
    if text.endswith(b"\n"):
        words = words[:-1]
    if text == b"":
        words = []
    s = Scheme.occurrence(LetterSet("etaoinshrdlcumwf"))
    with GpuFingerprintedDictionary.from_text(text, s) as d:
        assert d.size() == len(words)
        if words:
            with GpuFingerprintedDictionary(words, s) as ref:
                assert np.array_equal(d.prints_array(), ref.prints_array())
                for pat in (b"a", b"bc\r", b"", b"z"):
                    for m in (Metric.Hamming, Metric.Levenshtein):
                        assert d.query(pat, QueryOptions(m, 1)) == ref.query(pat, QueryOptions(m, 1))


def test_dictionary_from_text_config(oracle):
    """A config-2 dictionary built from its newline text on two shards equals
    the oracle (ids, stats), and the GPU byte histogram equals the host's."""
    from paper_1711_08475_b200 import compute_frequencies, compute_frequencies_gpu

    blob, offs, qblob, qoffs = _cfg_inputs(2, 120_000, 300)
    words = [bytes(blob[int(offs[i]):int(offs[i + 1])]) for i in range(len(offs) - 1)]
    text = b"\n".join(words) + b"\n"
    s = make_scheme(blob, Variant.Count, 16)
    assert np.array_equal(compute_frequencies_gpu(blob).counts, compute_frequencies(blob).counts)
    with GpuFingerprintedDictionary.from_text(text, s, devices=(0, 0)) as d:
        assert d.size() == len(words)
        csr, st = d.query_batch((qblob, qoffs), QueryOptions(Metric.Levenshtein, 1, True, True), True)
    assert_same(csr, st, *oracle.query_batch(blob, offs, qblob, qoffs, osch(s), Metric.Levenshtein, 1, True, True))


@pytest.mark.slow
@pytest.mark.parametrize("cfg,cell,nsample", [(3, 0, 40), (3, 1, 40), (4, 0, 40), (4, 1, 40), (5, 0, 40), (5, 5, 40)])
def test_full_size_configs_vs_oracle(oracle, cfg, cell, nsample):
    """BASELINE sizes (config 3: 2e6 words x 5e4 queries, config 4: 8e6 x 1e5,
    config 5: 6.4e7 x 1e6 on one GPU): the whole batch runs on the GPU; an
    evenly spaced query subsample is checked against the oracle (ids and
    QueryStats), plus the batch total against the filter-off run."""
    import bench
    w = bench.Workload(cfg, cell)  # the bench's workload: letters and query sources over the whole dictionary
    blob, offs, qblob, qoffs, scheme, metric = w.blob, w.offs, w.qblob, w.qoffs, w.scheme, w.metric
    nq = len(qoffs) - 1
    opt = QueryOptions(metric, 1, True, True)
    with GpuFingerprintedDictionary((blob, offs), scheme, keep_words=False) as d:
        csr, st = d.query_batch((qblob, qoffs), opt, per_query_stats=True)
    sb, so, idx = subsample(qblob, qoffs, max(1, nq // nsample))
    o_off, o_ids, o_st = oracle.query_batch(blob, offs, sb, so, osch(scheme), metric, 1, True, True)
    for j, q in enumerate(idx):
        assert np.array_equal(csr.row(q), o_ids[int(o_off[j]):int(o_off[j + 1])]), f"query {q}"
        assert np.array_equal(st[q], o_st[j]), f"stats of query {q}"
    assert int(st[:, 4].sum()) == len(csr.word_ids)


# ---------------------------------------------------------------- shard gathers

def test_device_csr_merge_equals_host_gather():
    """fpg_csr_merge_device over the shards' device-resident CSRs (the
    one-process-per-GPU gather, here with 3 shards on one GPU) equals the
    host gather of fpg_batch_download, and lifecycle errors are reported."""
    import torch

    from paper_1711_08475_b200.sharding import device_tensors, merge_device

    blob, offs, qblob, qoffs = _cfg_inputs(5, 60_000, 300)
    s = make_scheme(blob, Variant.Occurrence, 16)
    opt = QueryOptions(Metric.Levenshtein, 1, True, True)
    with GpuFingerprintedDictionary((blob, offs), s, devices=(0, 0, 0)) as d:
        b = d.batch()
        with pytest.raises(ValueError):  # run before upload: FPG_EINVAL, not a crash
            b.run(opt)
        with pytest.raises(ValueError):
            b.device_csr(0)
        b.upload(qblob, qoffs)
        b.run(opt, want_stats=True)
        host, _ = b.download()
        parts = [device_tensors(b.device_csr(i)) for i in range(3)]
        assert sum(int(p[1].numel()) for p in parts) == len(host.word_ids)
        m_off, m_ids = merge_device(parts, len(qoffs) - 1, 0)
        torch.cuda.synchronize()
        assert np.array_equal(m_off.cpu().numpy().view(np.uint64), host.offsets)
        assert np.array_equal(m_ids.cpu().numpy().view(np.uint32), host.word_ids)
        h = host_ms = b.host_ms()
        assert h["download_ms"] >= 0 and host_ms["assemble_ms"] >= 0


def _bench(args, env_extra=None, timeout=900):
    import os
    import subprocess
    import sys

    root = Path(__file__).resolve().parents[1]
    env = dict(os.environ, **(env_extra or {}))
    return subprocess.run([sys.executable, str(root / "bench.py"), *args], capture_output=True, text=True,
                          env=env, timeout=timeout, cwd=root)


def test_bench_gpus_n_one_process():
    """bench.py --gpus 2 without torchrun drives two shards from one process
    (here both on device 0 via FPG_BENCH_DEVICES) and reports n_gpus = 2 and
    the host gather cost inside e2e; without the override on a box with fewer
    GPUs it fails loudly."""
    import torch

    r = _bench(["--config", "1", "--gpus", "2", "--steps", "2", "--warmup", "1", "--no-cpu-baseline"],
               {"FPG_BENCH_DEVICES": "0,0"})
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["n_gpus"] == 2 and line["config"]["parallelism"] == "dict-shard x2"
    assert len(line["shard_ms_per_step"]) == 2 and line["e2e"]["gather_ms_per_step"] is not None
    if torch.cuda.device_count() < 3:
        r = _bench(["--config", "1", "--gpus", "3", "--steps", "1", "--warmup", "1", "--no-cpu-baseline"])
        assert r.returncode != 0 and "CUDA device" in (r.stderr + r.stdout)
