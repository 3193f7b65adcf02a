"""Generates tests/golden/reference_vectors.json by running the REFERENCE
itself (its header-only C++ library compiled from /root/reference into
oracle/_ref/libfpref.so by oracle/Makefile).  Re-run after changing the
inputs below:  python tests/golden/make_golden.py

The inputs are generated here with Python's `random` (seeded) and stored in
the fixture, so the fixture is self-contained: tests compare the oracle and
the GPU path against the reference's outputs without needing /root/reference.
"""
from __future__ import annotations

import hashlib
import json
import random
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
from oracle.oracle import Reference, pack  # noqa: E402

# The reference tests' letter sets (fingerprint_test.cpp:13-16) plus other
# parameterisations the reference accepts (b=4, p=4, p=5, mixed sets).
SCHEMES = [
    {"name": "occ16", "variant": 0, "letters": "etaoinshrdlcumwf", "b": 2, "p": 3},
    {"name": "halved8", "variant": 1, "letters": "etaoinsh", "b": 2, "p": 3},
    {"name": "count8", "variant": 2, "letters": "etaoinsh", "b": 2, "p": 3},
    {"name": "pos6", "variant": 3, "letters": "etaoin", "b": 2, "p": 3},
    {"name": "count4_b4", "variant": 2, "letters": "eaqz", "b": 4, "p": 3},
    {"name": "pos4_p4", "variant": 3, "letters": "abcd", "b": 2, "p": 4},
    {"name": "pos4_p5", "variant": 3, "letters": "xyza", "b": 2, "p": 5},
    {"name": "count16_b1", "variant": 2, "letters": "abcdefghijklmnop", "b": 1, "p": 3},
    {"name": "occ16_dense", "variant": 0, "letters": "abecdfghijklmnop", "b": 2, "p": 3},
]


def rand_word(rng: random.Random, lo: int, hi: int, alphabet: str) -> str:
    return "".join(rng.choice(alphabet) for _ in range(rng.randint(lo, hi)))


def main() -> None:
    ref = Reference()
    rng = random.Random(20240611)
    out: dict = {"generator": "tests/golden/make_golden.py", "source": "oracle/_ref/libfpref.so (reference headers)"}

    # 1. fingerprints of seeded words for each scheme, incl. empty/tiny/saturating strings
    words = ["", "e", "instance", "run", "ran", "eeee", "eee", "ee", "e" + "z" * 19, "zzzzzzze",
             "zzzzzze", "zzzzzzzz", "tea", "wof"]
    words += [rand_word(rng, 0, 24, "etaoinshrdlcumwfzyxq") for _ in range(1500)]
    words += [rand_word(rng, 0, 40, "abcdexyz\x00\xff") for _ in range(300)]
    blob, offs = pack(words)
    out["words"] = [w.encode("latin-1").hex() for w in words]
    out["schemes"] = []
    for s in SCHEMES:
        fps = ref.build_many(blob, offs, s["variant"], s["letters"], s["b"], s["p"])
        tab = ref.distance_table(s["variant"], s["letters"], s["b"], s["p"])
        rec = dict(s)
        rec["prints"] = [int(x) for x in fps]
        rec["distance_table_sha256"] = hashlib.sha256(tab.tobytes()).hexdigest()
        rec["distance_table_sample"] = {str(x): int(tab[x]) for x in range(0, 65536, 257)}
        rec["render_instance"] = ref.render(int(fps[2]), s["variant"], s["letters"], s["b"], s["p"])
        out["schemes"].append(rec)

    # 2. bounded verifiers vs the reference (k = 0..3)
    pairs = []
    base = ["", "a", "ab", "abc", "kitten", "sitting", "instance", "run", "ran", "short", "shorter"]
    for a in base:
        for b in base:
            pairs.append((a, b))
    for _ in range(600):
        a = rand_word(rng, 0, 12, "abc")
        if rng.random() < 0.5:
            b = list(a)
            for _ in range(rng.randint(0, 2)):
                op = rng.randint(0, 2)
                if op == 0 and b:
                    b[rng.randrange(len(b))] = rng.choice("abcd")
                elif op == 1:
                    b.insert(rng.randint(0, len(b)), rng.choice("abcd"))
                elif b:
                    del b[rng.randrange(len(b))]
            b = "".join(b)
        else:
            b = rand_word(rng, 0, 12, "abc")
        pairs.append((a, b))
    ver = []
    for a, b in pairs:
        rec = {"a": a, "b": b, "lev_full": ref.levenshtein_full(a, b)}
        rec["lev"] = [ref.levenshtein_bounded(a, b, k) for k in range(4)]
        rec["ham"] = [ref.hamming_bounded(a, b, k) for k in range(4)]
        ver.append(rec)
    out["verifiers"] = ver

    # 3. query_into over a small dictionary, all options, per-query stats
    dict_words = [rand_word(rng, 3, 9, "abcdefghijklmnop") for _ in range(1000)]
    dict_words += ["", "a", "ab", dict_words[0], dict_words[1]]  # empty, tiny, duplicates
    qwords = []
    for i in range(60):
        w = list(rng.choice(dict_words))
        if i % 3 == 1 and w:
            w[rng.randrange(len(w))] = rng.choice("abcdefghijklmnopq")
        elif i % 3 == 2:
            w.insert(rng.randint(0, len(w)), rng.choice("abcdefghijklmnop"))
        qwords.append("".join(w))
    qwords += ["", "a", "b", "abcdefghijklmnop" * 2]
    dblob, doffs = pack(dict_words)
    qblob, qoffs = pack(qwords)
    out["query_dict"] = [w.encode("latin-1").hex() for w in dict_words]
    out["query_patterns"] = [w.encode("latin-1").hex() for w in qwords]
    qres = []
    for s in SCHEMES[:4]:
        d = ref.dictionary(dblob, doffs, s["variant"], s["letters"], s["b"], s["p"])
        for metric in (0, 1):
            for k in (0, 1, 2, 3):
                for use_filter in (True, False):
                    for pre in (False, True):
                        if use_filter and not (metric == 0 or s["variant"] in (0, 2)):
                            continue
                        o, ids, st = d.query_batch(qblob, qoffs, metric, k, use_filter, pre, threads=4)
                        qres.append({"scheme": s["name"], "metric": metric, "k": k, "use_filter": use_filter,
                                     "length_prefilter": pre, "offsets": [int(x) for x in o],
                                     "ids": [int(x) for x in ids], "stats": st.astype(np.int64).tolist()})
        d.close()
    out["queries"] = qres

    # 4. letter selection on a skewed corpus
    corpus = np.frombuffer(("eeeeettttaaaooin" * 50 + "zqxj" + "".join(dict_words)).encode(), np.uint8)
    out["select_letters"] = {
        "corpus_sha256": hashlib.sha256(corpus.tobytes()).hexdigest(),
        "results": [{"count": c, "strategy": st, "letters": (ref.select_letters(corpus, c, st) or b"").hex()}
                    for c in (4, 6, 8, 16, 17, 30) for st in (0, 1, 2)],
    }

    path = Path(__file__).with_name("reference_vectors.json")
    path.write_text(json.dumps(out, separators=(",", ":")))
    print(f"wrote {path} ({path.stat().st_size} bytes)")


if __name__ == "__main__":
    main()
