"""K2's weight window is exact: the L1 distance between two fingerprints'
group weights never exceeds the reference's fingerprint distance F_D, so the
pairs K2 skips (distance > 2k) are pairs the reference rejects.

fp_gweight below restates the device function of the same name
(paper_1711_08475_b200/csrc/fpg_kernels.cuh); F_D comes from the oracle's
restatement of ComparisonTables (fingerprint.hpp:171-214).  CPU only.
"""
import random

import numpy as np
import pytest

from oracle.oracle import Oracle, oscheme, pack

ALPHABET = "etaoinshrdlcumwfgypbvkjxqz0123456789./:-_?=&%~ABCDEFGHIJKLMNOPQRSTUVW"

# (variant, width, b, p): occurrence 0, halved 1, count 2, position 3
CELLS = [(0, 16, 2, 3), (0, 32, 2, 3), (0, 64, 2, 3), (1, 16, 2, 3), (1, 32, 2, 3),
         (2, 16, 2, 3), (2, 32, 2, 3), (2, 64, 4, 3), (3, 16, 2, 3), (3, 32, 2, 3), (3, 64, 2, 3)]


def fp_gweight(fp: int, variant: int, width: int, b: int, p: int) -> list[int]:
    """Per-group count of "present" fields; field i goes to group i & 3."""
    g = [0, 0, 0, 0]
    if variant in (0, 1):
        for i in range(width):
            g[i & 3] += (fp >> i) & 1
        return g
    fw = b if variant == 2 else p
    nf = width // fw
    extra = 0 if variant == 2 else width - fw * nf
    fmask = (1 << fw) - 1
    for e in range(extra):
        g[e & 3] += (fp >> e) & 1
    for f in range(nf):
        v = (fp >> (width - fw * (f + 1))) & fmask
        g[(extra + f) & 3] += int(v != 0) if variant == 2 else int(v != fmask)
    return g


def _one_edit(w: str, rng: random.Random, alphabet: str) -> str:
    i = rng.randrange(len(w) + 1)
    op = rng.randrange(3)
    c = rng.choice(alphabet)
    if op == 0 and i < len(w):
        return w[:i] + c + w[i + 1:]
    if op == 1 and i < len(w) and len(w) > 1:
        return w[:i] + w[i + 1:]
    return w[:i] + c + w[i:]


@pytest.fixture(scope="module")
def oracle():
    return Oracle()


@pytest.mark.parametrize("variant,width,b,p", CELLS)
def test_group_weight_distance_bounds_fd(oracle, variant, width, b, p):
    cap = oracle.letter_capacity(variant, width, b, p)
    letters = ALPHABET[:cap]
    sch = oscheme(variant, letters, width, b, p)
    assert oracle.scheme_ok(sch)
    rng = random.Random(1000 * variant + width)
    alpha = ALPHABET[:max(cap + 6, 12)]
    words, pairs = [], []
    for _ in range(600):
        w = "".join(rng.choice(alpha) for _ in range(rng.randint(1, 40)))
        words.append(w)
        pairs.append(_one_edit(w, rng, alpha))                                     # near pair
        pairs.append("".join(rng.choice(alpha) for _ in range(rng.randint(1, 40))))  # random pair
    words = [w for w in words for _ in range(2)]
    fa = oracle.build_many(*pack(words), sch)
    fb = oracle.build_many(*pack(pairs), sch)
    tight = 0
    for x, y in zip(fa, fb):
        x, y = int(x), int(y)
        d = oracle.distance(x, y, sch)
        gx, gy = fp_gweight(x, variant, width, b, p), fp_gweight(y, variant, width, b, p)
        l1 = sum(abs(u - v) for u, v in zip(gx, gy))
        assert l1 <= d, (x, y, gx, gy, d)
        tight += l1 == d
    assert tight > 0  # the bound is reached, i.e. it is not vacuous


def test_group_weights_fit_the_sort_key():
    """k_weight_keys packs the group weights saturated at 15 below the length;
    saturation is 1-Lipschitz, so it can only coarsen the order."""
    rng = np.random.default_rng(0)
    a = rng.integers(0, 40, size=1000)
    b = rng.integers(0, 40, size=1000)
    assert np.all(np.abs(np.minimum(a, 15) - np.minimum(b, 15)) <= np.abs(a - b))
