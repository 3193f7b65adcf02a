"""The CPU oracle (oracle/fp_oracle.c) pinned against the reference: golden
vectors of the reference's own tests, fixtures produced by running the
reference (tests/golden/reference_vectors.json, made by make_golden.py), and
-- where oracle/_ref is built -- the reference library live.  Also the
generalised-width (W=32/64) properties the reference cannot pin."""
import hashlib
import json
import random
from pathlib import Path

import numpy as np
import pytest

from oracle.oracle import oscheme, pack

GOLD = json.loads((Path(__file__).parent / "golden" / "reference_vectors.json").read_text())
WORDS = [bytes.fromhex(h) for h in GOLD["words"]]


def osch(rec, width=16):
    return oscheme(rec["variant"], rec["letters"], width, rec["b"], rec["p"])


def test_instance_golden_renders(oracle):
    # fingerprint_test.cpp:60-66, acceptance_test.cpp:97-113
    want = ["1110111000010000", "01 10 01 00 10 11 10 00", "01 01 01 00 01 10 01 00", "111 011 100 111 000 1"]
    for rec, w in zip(GOLD["schemes"][:4], want):
        s = osch(rec)
        assert oracle.render(oracle.build("instance", s), s) == w


def test_tiny_and_saturation_goldens(oracle):
    occ, halved, count, pos = (osch(r) for r in GOLD["schemes"][:4])
    assert oracle.render(oracle.build("", pos), pos) == "111 111 111 111 111 0"      # fingerprint_test.cpp:73
    assert oracle.render(oracle.build("e", halved), halved) == "01 00 00 00 00 00 00 00"  # :75-76
    assert oracle.render(oracle.build("e" + "z" * 19, pos), pos) == "000 111 111 111 111 0"  # :83
    assert oracle.build("zzzzzzze", pos) == oracle.build("zzzzzzzz", pos)           # :85-87
    assert oracle.render(oracle.build("zzzzzze", pos), pos) == "110 111 111 111 111 0"  # :88
    assert oracle.render(oracle.build("eeee", count), count) == "11 00 00 00 00 00 00 00"  # :94
    assert oracle.render(oracle.build("eee", count), count) == "11 00 00 00 00 00 00 00"
    assert oracle.render(oracle.build("ee", count), count) == "10 00 00 00 00 00 00 00"


def test_distance_and_reject_goldens(oracle):
    occ = osch(GOLD["schemes"][0])
    run, ran = oracle.build("run", occ), oracle.build("ran", occ)
    assert oracle.distance(run, ran, occ) == 2 and not oracle.can_reject(run, ran, 1, occ)  # :194-225
    assert oracle.can_reject(oracle.build("tea", occ), oracle.build("wof", occ), 1, occ)
    count = osch(GOLD["schemes"][2])
    assert oracle.distance(oracle.build("eee", count), oracle.build("e", count), count) == 1
    # reference_test.cpp:61-72
    assert oracle.distance(0x1234, 0x1234, occ) == 0
    assert oracle.distance(0, 0b1010101010000000, occ) == 5
    assert oracle.distance(0, 0b0100000010000001, osch(GOLD["schemes"][3])) == 3


def test_capacities_and_validation(oracle):
    # fingerprint_test.cpp:30-48 (W = 16)
    assert oracle.letter_capacity(0, 16) == 16 and oracle.letter_capacity(1, 16) == 8
    assert oracle.letter_capacity(2, 16, 2) == 8 and oracle.letter_capacity(2, 16, 4) == 4
    assert oracle.letter_capacity(3, 16, 2, 3) == 6 and oracle.letter_capacity(3, 16, 2, 4) == 4
    assert oracle.letter_capacity(3, 16, 2, 5) == 4 and oracle.letter_capacity(2, 16, 3) == -1
    assert not oracle.scheme_ok(oscheme(0, "abc"))
    assert not oracle.scheme_ok(oscheme(1, "etaoinse"))  # duplicate letter
    # generalised widths
    assert oracle.letter_capacity(3, 64, 2, 3) == 22 and oracle.letter_capacity(2, 64, 4) == 16


@pytest.mark.parametrize("idx", range(len(GOLD["schemes"])))
def test_prints_match_reference_fixture(oracle, idx):
    rec = GOLD["schemes"][idx]
    blob, offs = pack(WORDS)
    assert [int(x) for x in oracle.build_many(blob, offs, osch(rec))] == rec["prints"]


@pytest.mark.parametrize("idx", range(len(GOLD["schemes"])))
def test_distance_table_matches_reference(oracle, idx):
    """All 2^16 xor values (fingerprint_test.cpp:156-192): field-by-field
    restatement == the reference's ComparisonTables."""
    rec = GOLD["schemes"][idx]
    s = osch(rec)
    tab = np.array([oracle.distance(x, 0, s) for x in range(65536)], np.uint8)
    assert hashlib.sha256(tab.tobytes()).hexdigest() == rec["distance_table_sha256"]


def test_verifiers_match_reference_fixture(oracle):
    for v in GOLD["verifiers"]:
        assert oracle.levenshtein_full(v["a"], v["b"]) == v["lev_full"]
        assert [oracle.levenshtein_bounded(v["a"], v["b"], k) for k in range(4)] == v["lev"]
        assert [oracle.hamming_bounded(v["a"], v["b"], k) for k in range(4)] == v["ham"]


def test_verifiers_exhaustive_abc(oracle):
    """edit_distance_test.cpp:47-111: bounded == full over {a,b,c}^<=4, k<=3."""
    words = [""]
    for L in range(1, 5):
        words += ["".join(t) for t in __import__("itertools").product("abc", repeat=L)]
    for a in words[::3]:
        for b in words:
            d = oracle.levenshtein_full(a, b)
            for k in range(4):
                assert oracle.levenshtein_bounded(a, b, k) == (d if d <= k else -1)
            if len(a) == len(b):
                h = oracle.hamming_full(a, b)
                for k in range(4):
                    assert oracle.hamming_bounded(a, b, k) == (h if h <= k else -1)


@pytest.mark.parametrize("case", range(len(GOLD["queries"])))
def test_query_batch_matches_reference_fixture(oracle, case):
    q = GOLD["queries"][case]
    rec = next(r for r in GOLD["schemes"] if r["name"] == q["scheme"])
    dblob, doffs = pack([bytes.fromhex(h) for h in GOLD["query_dict"]])
    qblob, qoffs = pack([bytes.fromhex(h) for h in GOLD["query_patterns"]])
    off, ids, st = oracle.query_batch(dblob, doffs, qblob, qoffs, osch(rec), q["metric"], q["k"],
                                      q["use_filter"], q["length_prefilter"], threads=2)
    assert [int(x) for x in off] == q["offsets"]
    assert [int(x) for x in ids] == q["ids"]
    assert st.astype(np.int64).tolist() == q["stats"]


def test_unsupported_metric_raises(oracle):
    dblob, doffs = pack(["abcdef"])
    qblob, qoffs = pack(["abcdef"])
    with pytest.raises(ValueError):
        oracle.query_batch(dblob, doffs, qblob, qoffs, oscheme(3, "abcdef"), 1, 1, True, False)


def test_select_letters_matches_reference_fixture(oracle):
    sl = GOLD["select_letters"]
    corpus = np.frombuffer(("eeeeettttaaaooin" * 50 + "zqxj" + "".join(
        bytes.fromhex(h).decode("latin-1") for h in GOLD["query_dict"])).encode(), np.uint8)
    assert hashlib.sha256(corpus.tobytes()).hexdigest() == sl["corpus_sha256"]
    for r in sl["results"]:
        got = oracle.select_letters(corpus, r["count"], r["strategy"])
        assert (got or b"").hex() == r["letters"]


# ---------------------------------------------------------------- generalised widths (unpinned by the reference)

def _rand(rng, lo, hi, alpha="abcdefghijklmnopqrstuvwxyz"):
    return "".join(rng.choice(alpha) for _ in range(rng.randint(lo, hi)))


@pytest.mark.parametrize("variant,width,b,p", [(0, 32, 2, 3), (0, 64, 2, 3), (1, 32, 2, 3), (1, 64, 2, 3),
                                               (2, 32, 2, 3), (2, 64, 4, 3), (3, 32, 2, 3), (3, 64, 2, 3)])
def test_wide_schemes_soundness_and_growth(oracle, variant, width, b, p):
    """acceptance_test.cpp:117-215 restated at W: ceil(F_D/2) <= distance
    and one edit changes F_D by at most 2."""
    cap = oracle.letter_capacity(variant, width, b, p)
    alphabet = [chr(c) for c in range(33, 33 + max(cap + 4, 30))]
    rng = random.Random(width * 31 + variant)
    letters = "".join(rng.sample(alphabet, cap))
    s = oscheme(variant, letters, width, b, p)
    for _ in range(1500):
        a = _rand(rng, 0, 20, alphabet)
        bb = _rand(rng, len(a), len(a), alphabet)
        fa, fb = oracle.build(a, s), oracle.build(bb, s)
        assert (oracle.distance(fa, fb, s) + 1) // 2 <= oracle.hamming_full(a, bb)
        if variant in (0, 2):
            c = _rand(rng, 0, 20, alphabet)
            assert (oracle.distance(fa, oracle.build(c, s), s) + 1) // 2 <= oracle.levenshtein_full(a, c)
        if a:
            sub = list(a)
            sub[rng.randrange(len(a))] = rng.choice(alphabet)
            assert oracle.distance(oracle.build("".join(sub), s), fb, s) <= oracle.distance(fa, fb, s) + 2


def test_wide_occurrence_matches_membership(oracle):
    rng = random.Random(5)
    alphabet = [chr(c) for c in range(40, 104)]
    s = oscheme(0, "".join(alphabet), 64)
    for _ in range(300):
        w = _rand(rng, 0, 30, alphabet)
        f = oracle.build(w, s)
        for q, c in enumerate(alphabet):
            assert ((f >> (63 - q)) & 1) == (c in w)
