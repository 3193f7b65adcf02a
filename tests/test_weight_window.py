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


GROUPS = 8  # kGroups in fpg_kernels.cuh


def fp_gweight(fp: int, variant: int, width: int, b: int, p: int) -> list[int]:
    """Per-group count of "present" fields; field i goes to group i & 7."""
    g = [0] * GROUPS
    if variant in (0, 1):
        for i in range(width):
            g[i % GROUPS] += (fp >> i) & 1
        return g
    fw = b if variant == 2 else p
    nf = width // fw
    extra = 0 if variant == 2 else width - fw * nf
    fmask = (1 << fw) - 1
    for e in range(extra):
        g[e % GROUPS] += (fp >> e) & 1
    for f in range(nf):
        v = (fp >> (width - fw * (f + 1))) & fmask
        g[(extra + f) % GROUPS] += int(v != 0) if variant == 2 else int(v != fmask)
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


@pytest.mark.parametrize("variant,width,b,p", CELLS)
def test_group_weights_fit_a_nibble(oracle, variant, width, b, p):
    """Group weights travel as 8 nibbles (sort key, slab boxes, K2's window):
    no group can hold more than 15 present fields at W <= 64."""
    cap = oracle.letter_capacity(variant, width, b, p)
    sch = oscheme(variant, ALPHABET[:cap], width, b, p)
    fp = (1 << width) - 1 if variant != 3 else 0  # every field present (position: all-zero fields)
    assert max(fp_gweight(fp, variant, width, b, p)) <= 15
