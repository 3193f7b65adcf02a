"""The C restatement vs the reference library itself (oracle/_ref, compiled
from /root/reference headers) on fresh random inputs, all four variants and
both metrics at W=16.  Skipped where oracle/_ref was never built."""
import random

import numpy as np
import pytest

from oracle.oracle import oscheme, pack

SCHEMES = [(0, "etaoinshrdlcumwf", 2, 3), (1, "etaoinsh", 2, 3), (2, "etaoinsh", 2, 3), (3, "etaoin", 2, 3),
           (2, "eaqz", 4, 3), (3, "xyza", 2, 5)]


def _words(seed, n, lo=0, hi=14, alpha="etaoinshrdlcumwfxyzq"):
    rng = random.Random(seed)
    return ["".join(rng.choice(alpha) for _ in range(rng.randint(lo, hi))) for _ in range(n)]


@pytest.mark.parametrize("variant,letters,b,p", SCHEMES)
def test_build_matches_reference(oracle, reference, variant, letters, b, p):
    blob, offs = pack(_words(variant * 7 + b, 20000, 0, 40))
    ours = oracle.build_many(blob, offs, oscheme(variant, letters, 16, b, p))
    ref = reference.build_many(blob, offs, variant, letters, b, p).astype(np.uint64)
    assert np.array_equal(ours, ref)


@pytest.mark.parametrize("variant,letters,b,p", SCHEMES[:4])
@pytest.mark.parametrize("metric", [0, 1])
@pytest.mark.parametrize("pre", [False, True])
def test_query_batch_matches_reference(oracle, reference, variant, letters, b, p, metric, pre):
    if metric == 1 and variant in (1, 3):
        pytest.skip("halved/position do not filter Levenshtein (fingerprint.hpp:36-38)")
    dwords = _words(11 + variant, 3000, 2, 10)
    rng = random.Random(variant)
    qwords = [rng.choice(dwords) if i % 2 else _words(i, 1, 2, 10)[0] for i in range(120)]
    dblob, doffs = pack(dwords)
    qblob, qoffs = pack(qwords)
    o = oracle.query_batch(dblob, doffs, qblob, qoffs, oscheme(variant, letters, 16, b, p), metric, 1, True, pre, 4)
    d = reference.dictionary(dblob, doffs, variant, letters, b, p)
    r = d.query_batch(qblob, qoffs, metric, 1, True, pre, 4)
    for x, y in zip(o, r):
        assert np.array_equal(x, y)


def test_select_letters_matches_reference(oracle, reference):
    rng = np.random.default_rng(3)
    for _ in range(20):
        corpus = rng.integers(97, 97 + rng.integers(10, 26), 5000).astype(np.uint8)
        for count in (4, 8, 16):
            for strat in (0, 1, 2):
                assert oracle.select_letters(corpus, count, strat) == reference.select_letters(corpus, count, strat)
