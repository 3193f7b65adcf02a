"""Host-side checks that need no GPU: the C-ABI library loads and exports
every symbol include/fpg.h declares, the reference-mirror API's host logic
(scheme layout, validation errors, rendering, letter selection), the seeded
generators, and that the product never reaches the oracle."""
import ast
import ctypes
import re
from pathlib import Path

import numpy as np
import pytest

from paper_1711_08475_b200 import (LetterSet, LetterStrategy, Metric, Scheme, Variant, compute_frequencies,
                                   english_default_letters, pack_strings, render, select_letters,
                                   variant_supports)
from paper_1711_08475_b200._lib import FPG_SIGNATURES, load_fpg
from paper_1711_08475_b200.corpus import CELLS, CONFIGS, generate_dictionary, generate_queries, subsample
from paper_1711_08475_b200.sharding import merge_csr, shard_bounds

ROOT = Path(__file__).resolve().parents[1]


def header_symbols():
    text = (ROOT / "include" / "fpg.h").read_text()
    return sorted(set(re.findall(r"\b(fpg_[a-z_]+)\s*\(", text)))


def test_library_exports_every_header_symbol():
    lib = load_fpg()
    syms = header_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(lib, s), f"libfpg.so does not export {s}"
    assert set(syms) == set(FPG_SIGNATURES), "ctypes table out of sync with include/fpg.h"
    assert lib.fpg_abi_version() == 3


def test_python_capacity_equals_c_abi():
    # Scheme.letter_capacity is host arithmetic (no libfpg.so load, so the
    # reference arm of bench.py never maps the CUDA library); it must agree
    # with fpg_letter_capacity on every parameterisation
    from paper_1711_08475_b200.fingerprints import _letter_capacity

    lib = load_fpg()
    for v in range(5):
        for w in (8, 16, 24, 32, 64, 128):
            for b in range(-1, 9):
                for p in range(-1, 70, 3):
                    c = lib.fpg_letter_capacity(v, w, b, p)
                    assert _letter_capacity(v, w, b, p) == (c if c >= 0 else -1), (v, w, b, p)


def test_library_is_sm100a_cuda():
    out = __import__("subprocess").run(["cuobjdump", "--list-elf", str(ROOT / "paper_1711_08475_b200/lib/libfpg.so")],
                                       capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_no_device_is_reported_cleanly():
    n = ctypes.c_int(-1)
    code = load_fpg().fpg_device_count(ctypes.byref(n))
    assert code in (0, -3)


def test_scheme_capacity_and_errors():
    # fingerprint_test.cpp:30-48
    assert Scheme.letter_capacity(Variant.Occurrence) == 16
    assert Scheme.letter_capacity(Variant.OccurrenceHalved) == 8
    assert Scheme.letter_capacity(Variant.Count, 2) == 8 and Scheme.letter_capacity(Variant.Count, 4) == 4
    assert Scheme.letter_capacity(Variant.Position, 2, 3) == 6
    assert Scheme.letter_capacity(Variant.Position, 2, 5) == 4
    assert Scheme.letter_capacity(Variant.Position, 2, 3, 64) == 22
    with pytest.raises(ValueError):
        Scheme.letter_capacity(Variant.Count, 3)
    with pytest.raises(ValueError):
        Scheme.occurrence(LetterSet("abc"))
    with pytest.raises(ValueError):
        LetterSet("aba")
    pos = Scheme.position(LetterSet("etaoin"), 3)
    assert pos.position_slots() == 5 and pos.extra_occurrence_slots() == 1 and pos.field_count() == 6
    assert pos.field_width(0) == 3 and pos.field_width(5) == 1
    assert [pos.field_shift(i) for i in range(6)] == [13, 10, 7, 4, 1, 0]
    assert variant_supports(Variant.Count, Metric.Levenshtein)
    assert not variant_supports(Variant.Position, Metric.Levenshtein)
    assert not variant_supports(Variant.OccurrenceHalved, Metric.Levenshtein)


def test_c_abi_scheme_validation():
    lib = load_fpg()
    ok = Scheme.count(LetterSet("etaoinsh")).c_struct()
    assert lib.fpg_scheme_validate(ctypes.byref(ok)) == 0
    bad = Scheme.count(LetterSet("etaoinsh")).c_struct()
    bad.nletters = 7
    assert lib.fpg_scheme_validate(ctypes.byref(bad)) == -1
    dup = Scheme.occurrence(LetterSet("etaoinshrdlcumwf")).c_struct()
    dup.letters[3] = dup.letters[0]
    assert lib.fpg_scheme_validate(ctypes.byref(dup)) == -1
    assert lib.fpg_scheme_supports(ctypes.byref(ok), 1) == 1


def test_render_matches_oracle(oracle):
    from oracle.oracle import oscheme
    rng = np.random.default_rng(0)
    for v, w, b, p in [(0, 16, 2, 3), (1, 32, 2, 3), (2, 64, 4, 3), (3, 64, 2, 3), (3, 16, 2, 5)]:
        cap = Scheme.letter_capacity(Variant(v), b, p, w)
        letters = bytes(range(40, 40 + cap))
        s = Scheme.make(Variant(v), LetterSet(letters), b, p, w)
        o = oscheme(v, letters, w, b, p)
        for _ in range(50):
            f = int(rng.integers(0, 2 ** 63)) & ((1 << w) - 1)
            assert render(f, s) == oracle.render(f, o)


def test_select_letters_matches_oracle(oracle):
    rng = np.random.default_rng(1)
    for _ in range(20):
        blob = rng.integers(97, 123, 3000).astype(np.uint8)
        for count in (4, 8, 16):
            for st in LetterStrategy:
                got = select_letters(compute_frequencies(blob), count, st).symbols()
                assert got == oracle.select_letters(blob, count, int(st))
    with pytest.raises(ValueError):
        select_letters(compute_frequencies(b"abc"), 4, LetterStrategy.Common)
    assert english_default_letters().startswith("etaoin")


def test_pack_strings_roundtrip():
    words = [b"", b"a", "bc", b"\x00\xff"]
    blob, offs = pack_strings(words)
    assert offs.tolist() == [0, 0, 1, 3, 5]
    assert bytes(blob) == b"abc\x00\xff"


@pytest.mark.parametrize("cfg", [1, 2, 3, 4, 5])
def test_generators_deterministic_and_prefix_stable(cfg):
    a_blob, a_off = generate_dictionary(cfg, n=5000)
    b_blob, b_off = generate_dictionary(cfg, n=5000, threads=3)
    assert np.array_equal(a_blob, b_blob) and np.array_equal(a_off, b_off)
    c_blob, c_off = generate_dictionary(cfg, n=2000, first=3000)  # shard of the same stream
    assert np.array_equal(a_blob[int(a_off[3000]):], c_blob)
    lens = np.diff(a_off.astype(np.int64))
    lo, hi = {1: (4, 16), 2: (4, 20), 3: (2, 24), 4: (20, 100), 5: (4, 16)}[cfg]
    assert lens.min() >= lo and lens.max() <= hi
    q1, o1 = generate_queries(cfg, a_blob, a_off, nq=300)
    q2, o2 = generate_queries(cfg, a_blob, a_off, nq=300)
    assert np.array_equal(q1, q2) and np.array_equal(o1, o2)


def test_generator_query_kinds():
    """Config 1: even queries are dictionary words with exactly one substitution."""
    blob, off = generate_dictionary(1, n=20000)
    words = {bytes(blob[int(off[i]):int(off[i + 1])]) for i in range(20000)}
    qb, qo = generate_queries(1, blob, off, nq=200)
    qs = [bytes(qb[int(qo[i]):int(qo[i + 1])]) for i in range(200)]
    for q in qs[::2]:
        assert q not in words or any(sum(x != y for x, y in zip(q, w)) == 1 for w in words if len(w) == len(q))
    # config 3 realised mean length ~8 (BASELINE.json:9)
    b3, o3 = generate_dictionary(3, n=200000)
    assert 7.7 < np.diff(o3.astype(np.int64)).mean() < 8.3


def test_cells_are_feasible_and_sound():
    for cfg, cells in CELLS.items():
        for v, w, b, p, m in cells:
            assert variant_supports(v, m), (cfg, v, m)
            cap = Scheme.letter_capacity(v, b, p, w)
            sigma = 46 if cfg == 4 else 26
            assert cap <= sigma, (cfg, v, w)
    assert CONFIGS[5].n_words == 64_000_000


def test_shard_bounds_and_merge():
    assert [shard_bounds(10, 3, r) for r in range(3)] == [(0, 3), (3, 6), (6, 10)]
    a = (np.array([0, 1, 1, 3], np.uint64), np.array([0, 1, 2], np.uint32))
    b = (np.array([0, 0, 2, 3], np.uint64), np.array([5, 6, 7], np.uint32))
    off, ids = merge_csr([a, b])
    assert off.tolist() == [0, 1, 3, 6] and ids.tolist() == [0, 5, 6, 1, 2, 7]


def test_subsample():
    qb, qo = pack_strings(["a", "bb", "ccc", "dddd", "e"])
    b, o, idx = subsample(qb, qo, 2)
    assert idx.tolist() == [0, 2, 4] and bytes(b) == b"accce"


def test_cpp_reference_extension_host(tmp_path):
    """include/fingerprints/b200_ref.hpp compiles in ONE translation unit with
    the reference's corpus.hpp, dictionary.hpp and reference.hpp (no type
    collision), and the reference-side pair test it exposes agrees with
    reference.hpp's field-by-field distance."""
    import subprocess

    from conftest import REF_INCLUDE, build_api_check_ref

    if not (REF_INCLUDE / "fingerprints" / "dictionary.hpp").exists():
        pytest.skip("reference headers absent")
    exe = build_api_check_ref(tmp_path / "api_check_ref")
    out = subprocess.run([str(exe), "host"], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr + out.stdout
    assert "api_check_ref host: ok" in out.stdout


def test_product_never_imports_the_oracle():
    """Only tests/, smoke() and bench.py's CPU legs may touch oracle/."""
    for path in (ROOT / "paper_1711_08475_b200").rglob("*.py"):
        tree = ast.parse(path.read_text())
        for node in ast.walk(tree):
            if isinstance(node, ast.ImportFrom):
                assert not (node.module or "").startswith("oracle"), path
            if isinstance(node, ast.Import):
                assert not any(a.name.startswith("oracle") for a in node.names), path
    for path in (ROOT / "paper_1711_08475_b200" / "csrc").rglob("*"):
        if path.is_file():
            assert "fp_oracle" not in path.read_text(errors="ignore"), path


def test_cpp_drop_in_headers_compile_and_host_logic(tmp_path):
    """Reference-style C++ caller code compiles against include/fingerprints/
    and its host-side logic (Scheme, LetterSet, render, errors) holds."""
    import subprocess

    from conftest import build_api_check

    exe = build_api_check(tmp_path)
    out = subprocess.run([str(exe), "host"], capture_output=True, text=True, check=True).stdout
    assert "api_check host: ok" in out
