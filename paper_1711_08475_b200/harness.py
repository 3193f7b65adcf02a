"""GPU-backed benchmark harness: the reference's `run_benchmark`,
`emit_figure_data` and report formats on libfpg.so.

Mirrors /root/reference/proj/include/fingerprints/bench.hpp and report.hpp:

* ``BenchConfig`` / ``BenchReport`` (bench.hpp:15-57): same fields and meaning.
* ``run_benchmark`` (bench.hpp:97-180): it selects letters over the whole
  collection and builds the scheme. It times construction. It then times one
  filter-off pass ("naive", T_n) and one filter-on pass (T_f) over the same
  queries. If the two match counts differ it raises (``logic_error``, here
  ``RuntimeError``). Speedup is T_n / T_f, and rejection % is
  rejected_by_fingerprint / (compared - rejected_by_length).
* ``emit_figure_data`` (bench.hpp:207-253): per word size, one naive row and
  one row per (variant, strategy).
* ``bench_csv_header`` / ``to_csv_row`` / ``to_text`` / ``to_json_line`` /
  ``sweep_csv_header`` (report.hpp:14-102): same columns and precision.

What differs from the reference, by design:

* A "pass" is one GPU batch (``fpg_batch_run``): every query against every word.
  The naive pass sets ``exhaustive``: no fingerprint or sig' pruning at all, every
  length-compatible pair goes to the byte verifier (the GPU's own naive scan).
  Time is the CUDA-event device time of the batch, query fingerprinting included
  (the reference times ``query_into`` calls, which fingerprint the pattern,
  dictionary.hpp:84).
* ``generate_synthetic`` and ``sample_queries`` keep the reference's semantics
  (corpus.hpp:44-112): fixed-length i.i.d. words from a frequency table;
  queries drawn with replacement and distorted by up to ``max_errors``
  substitutions, each applied with probability 0.5. They draw from numpy's
  seeded PCG64 rather than ``std::mt19937_64`` with implementation-defined
  ``std::discrete_distribution``, so the corpora are deterministic but not
  byte-identical to the reference's. Parity tests therefore feed both sides
  the same words.
"""
from __future__ import annotations

import argparse
import json
import sys
from dataclasses import dataclass, field
from typing import Sequence

import numpy as np

from .fingerprints import (GpuFingerprintedDictionary, LetterStrategy, Metric, QueryOptions, QueryStats, Scheme,
                           Variant, compute_frequencies, english_letter_frequencies, pack_strings, select_letters)

_VARIANT_NAME = {Variant.Occurrence: "occurrence", Variant.OccurrenceHalved: "occurrence-halved",
                 Variant.Count: "count", Variant.Position: "position"}
_STRATEGY_NAME = {LetterStrategy.Common: "common", LetterStrategy.Mixed: "mixed", LetterStrategy.Rare: "rare"}
_METRIC_NAME = {Metric.Hamming: "hamming", Metric.Levenshtein: "levenshtein"}


@dataclass
class BenchConfig:
    """bench.hpp:15-31 (plus the B200 width and device)."""

    dataset: str = "unnamed"
    words: Sequence = ()
    variant: Variant = Variant.Occurrence
    strategy: LetterStrategy = LetterStrategy.Common
    metric: Metric = Metric.Hamming
    k: int = 1
    bits_per_count: int = 2
    bits_per_position: int = 3
    query_count: int = 1000
    iterations: int = 100
    distort_max_errors: int = 0
    seed: int = 0
    levenshtein_length_prefilter: bool = False
    queries_override: Sequence | None = None
    word_length: int = 0
    width: int = 16
    device: int = 0


@dataclass
class BenchReport:
    """bench.hpp:33-57."""

    dataset: str = ""
    variant: Variant = Variant.Occurrence
    strategy: LetterStrategy = LetterStrategy.Common
    metric: Metric = Metric.Hamming
    k: int = 1
    word_length: int = 0
    word_count: int = 0
    letters: str = ""
    t_naive_ns: float = 0.0
    t_fingerprint_ns: float = 0.0
    speedup: float = 0.0
    rejection_pct: float = 0.0
    construction_mbps: float = 0.0
    matches_naive: int = 0
    matches_fingerprint: int = 0
    filtered_stats: QueryStats = field(default_factory=QueryStats)
    query_count: int = 0
    iterations: int = 0
    seed: int = 0
    environment: str = ""


@dataclass
class SweepConfig:
    """bench.hpp:182-197."""

    word_sizes: Sequence[int] = ()
    corpus_bytes: int = 256 * 1024
    variants: Sequence[Variant] = (Variant.Occurrence, Variant.Count, Variant.Position)
    strategies: Sequence[LetterStrategy] = (LetterStrategy.Common, LetterStrategy.Mixed, LetterStrategy.Rare)
    metric: Metric = Metric.Hamming
    k: int = 1
    bits_per_count: int = 2
    bits_per_position: int = 3
    query_count: int = 200
    iterations: int = 1
    distort_max_errors: int = 0
    seed: int = 0
    device: int = 0


@dataclass
class SweepRow:
    """bench.hpp:199-204."""

    word_size: int = 0
    variant: str = ""
    strategy: str = ""
    mean_pair_ns: float = 0.0


# ---------------------------------------------------------------- corpora

def generate_synthetic(total_bytes: int, word_length: int, frequencies, seed: int) -> list[bytes]:
    """corpus.hpp:44-70: fixed-length words, symbols i.i.d. from `frequencies`
    ((symbol, weight) pairs), until at least `total_bytes` bytes exist."""
    if word_length <= 0:
        raise ValueError("generate_synthetic: word length must be positive")
    freqs = list(frequencies)
    if not freqs:
        raise ValueError("generate_synthetic: empty distribution")
    symbols = np.array([s if isinstance(s, int) else ord(s) for s, _ in freqs], dtype=np.uint8)
    w = np.array([float(x) for _, x in freqs])
    n = -(-int(total_bytes) // word_length) if total_bytes > 0 else 0
    rng = np.random.default_rng(seed)
    picks = rng.choice(len(symbols), size=(n, word_length), p=w / w.sum())
    return [bytes(row) for row in symbols[picks]]


def sample_queries(words: Sequence, n: int, max_errors: int = 0, error_probability: float = 0.5,
                   seed: int = 0) -> list[bytes]:
    """corpus.hpp:80-112: n words drawn uniformly with replacement, each with
    up to max_errors substitutions (each applied with error_probability) at a
    uniform position, by a uniform symbol of the corpus alphabet."""
    if not words:
        raise ValueError("sample_queries: empty word list")
    ws = [w if isinstance(w, bytes) else bytes(w, "latin-1") for w in words]
    alphabet = sorted(set(b"".join(ws)))
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(n):
        q = bytearray(ws[int(rng.integers(len(ws)))])
        for _ in range(max_errors):
            if q and rng.random() < error_probability:
                q[int(rng.integers(len(q)))] = alphabet[int(rng.integers(len(alphabet)))]
        out.append(bytes(q))
    return out


# ---------------------------------------------------------------- timing

def _pass(batch, opt: QueryOptions, iterations: int):
    """`iterations` timed GPU batches; returns (device ns, QueryStats of one
    pass, matches of one pass).  Like run_pass (bench.hpp:80-90) every timed
    batch collects QueryStats; an untimed batch with the same options comes
    first, so the timed ones reuse its tile plan and the stats and matches
    are read outside the timed region."""
    batch.run(opt, want_stats=True)
    csr, st = batch.download()
    matches = int(csr.offsets[-1])
    s = st.sum(axis=0) if len(st) else np.zeros(5, np.uint64)
    stats = QueryStats(*(int(x) for x in s))
    total_ns = 0.0
    for _ in range(iterations):
        batch.run(opt, want_stats=True)
        total_ns += batch.timing()["run_ms"] * 1e6
    return total_ns, stats, matches


def run_benchmark(config: BenchConfig) -> BenchReport:
    """bench.hpp:97-180 on the GPU."""
    words = config.words
    n_words = (len(words[1]) - 1) if isinstance(words, tuple) else len(words)
    if n_words == 0:
        raise ValueError("run_benchmark: empty dictionary")
    if config.query_count < 1 or config.iterations < 1 or config.k < 1:
        raise ValueError("run_benchmark: query_count, iterations and k must be >= 1")
    blob, offs = words if isinstance(words, tuple) else pack_strings(words)
    cap = Scheme.letter_capacity(config.variant, config.bits_per_count, config.bits_per_position, config.width)
    letters = select_letters(compute_frequencies(blob), cap, config.strategy)
    scheme = Scheme.make(config.variant, letters, config.bits_per_count, config.bits_per_position, config.width)
    if not scheme.supports(config.metric):
        raise ValueError(f"{_VARIANT_NAME[config.variant]} fingerprints do not filter for the "
                         f"{_METRIC_NAME[config.metric]} distance")
    word_bytes = int(offs[-1] - offs[0])
    if config.queries_override is not None:
        queries = list(config.queries_override)
    else:
        word_list = [bytes(blob[int(offs[i]):int(offs[i + 1])]) for i in range(n_words)]
        queries = sample_queries(word_list, config.query_count, config.distort_max_errors, 0.5, config.seed)
    qblob, qoffs = pack_strings(queries)

    # construction is timed on a warm context (the first dictionary of a
    # process also pays CUDA context and module set-up)
    GpuFingerprintedDictionary((blob, offs), scheme, devices=(config.device,), keep_words=False).close()
    with GpuFingerprintedDictionary((blob, offs), scheme, devices=(config.device,), keep_words=False) as d:
        construction_s = d.build_seconds()
        batch = d.batch()
        batch.upload(qblob, qoffs)
        batch.run(QueryOptions(config.metric, config.k, True, config.levenshtein_length_prefilter))  # warm-up
        naive_ns, _, naive_matches = _pass(
            batch, QueryOptions(config.metric, config.k, False, config.levenshtein_length_prefilter, exhaustive=True),
            config.iterations)
        filt_ns, fstats, filt_matches = _pass(
            batch, QueryOptions(config.metric, config.k, True, config.levenshtein_length_prefilter),
            config.iterations)
        batch.close()
    if naive_matches != filt_matches:
        raise RuntimeError(f"filter dropped matches: naive {naive_matches} vs filtered {filt_matches}")

    pairs = float(config.iterations) * len(queries) * n_words
    r = BenchReport(dataset=config.dataset, variant=config.variant, strategy=config.strategy, metric=config.metric,
                    k=config.k, word_length=config.word_length, word_count=n_words,
                    letters=scheme.letters().symbols().decode("latin-1"), query_count=len(queries),
                    iterations=config.iterations, seed=config.seed, environment=_environment(config.device))
    r.t_naive_ns = naive_ns / pairs
    r.t_fingerprint_ns = filt_ns / pairs
    r.speedup = r.t_naive_ns / r.t_fingerprint_ns if r.t_fingerprint_ns > 0 else 0.0
    pool = fstats.compared - fstats.rejected_by_length
    r.rejection_pct = 0.0 if pool == 0 else 100.0 * fstats.rejected_by_fingerprint / pool
    r.construction_mbps = word_bytes / 1e6 / construction_s if construction_s > 0 else 0.0
    r.matches_naive = naive_matches
    r.matches_fingerprint = filt_matches
    r.filtered_stats = fstats
    return r


def emit_figure_data(config: SweepConfig) -> list[SweepRow]:
    """bench.hpp:207-253: per-pair time over synthetic English words, one row
    per (word size, variant, strategy) plus a naive row per size."""
    if not config.word_sizes:
        raise ValueError("emit_figure_data: no word sizes")
    rows = []
    for size in config.word_sizes:
        words = generate_synthetic(config.corpus_bytes, size, english_letter_frequencies(), config.seed)
        queries = sample_queries(words, config.query_count, config.distort_max_errors, 0.5, config.seed)
        blob, offs = pack_strings(words)
        qblob, qoffs = pack_strings(queries)
        freq = compute_frequencies(blob)
        pairs = float(config.iterations) * len(queries) * len(words)

        def timed(scheme, use_filter):
            with GpuFingerprintedDictionary((blob, offs), scheme, devices=(config.device,), keep_words=False) as d:
                b = d.batch()
                b.upload(qblob, qoffs)
                opt = QueryOptions(config.metric, config.k, use_filter, False, exhaustive=not use_filter)
                b.run(opt)  # warm-up
                ns, _, _ = _pass(b, opt, config.iterations)
                b.close()
            return ns / pairs

        # the naive path ignores fingerprints, so any scheme will do (bench.hpp:224-231)
        rows.append(SweepRow(size, "naive", "-",
                             timed(Scheme.occurrence(select_letters(freq, 16, LetterStrategy.Common)), False)))
        for v in config.variants:
            cap = Scheme.letter_capacity(v, config.bits_per_count, config.bits_per_position)
            for s in config.strategies:
                scheme = Scheme.make(v, select_letters(freq, cap, s), config.bits_per_count, config.bits_per_position)
                rows.append(SweepRow(size, _VARIANT_NAME[v], _STRATEGY_NAME[s], timed(scheme, True)))
    return rows


def _environment(device: int) -> str:
    try:
        import torch

        return f"{torch.cuda.get_device_name(device)}, libfpg.so (sm_100a)"
    except Exception:  # environment string only
        return "libfpg.so (sm_100a)"


# ---------------------------------------------------------------- reports (report.hpp)

def bench_csv_header() -> str:
    """report.hpp:14-17."""
    return ("dataset,variant,strategy,metric,k,word_length,T_n_ns,T_f_ns,speedup,"
            "rejection_pct,construction_mbps,matches")


def sweep_csv_header() -> str:
    """report.hpp:85-87."""
    return "word_size,variant,strategy,mean_pair_ns"


def to_csv_row(r) -> str:
    """report.hpp:19-27 (BenchReport) and :89-94 (SweepRow)."""
    if isinstance(r, SweepRow):
        return f"{r.word_size},{r.variant},{r.strategy},{r.mean_pair_ns:.3f}"
    return (f"{r.dataset},{_VARIANT_NAME[r.variant]},{_STRATEGY_NAME[r.strategy]},{_METRIC_NAME[r.metric]},{r.k},"
            f"{r.word_length},{r.t_naive_ns:.3f},{r.t_fingerprint_ns:.3f},{r.speedup:.3f},"
            f"{r.rejection_pct:.2f},{r.construction_mbps:.2f},{r.matches_fingerprint}")


def to_text(r: BenchReport) -> str:
    """report.hpp:29-54."""
    fs = r.filtered_stats
    head = f"dataset:            {r.dataset} ({r.word_count} words"
    if r.word_length:
        head += f", length {r.word_length}"
    return "\n".join([
        head + ")",
        f"scheme:             {_VARIANT_NAME[r.variant]} / {_STRATEGY_NAME[r.strategy]}, letters \"{r.letters}\"",
        f"query:              {_METRIC_NAME[r.metric]}, k={r.k}, {r.query_count} queries x {r.iterations} "
        f"iterations, seed {r.seed}",
        f"naive time/pair:    {r.t_naive_ns:.3f} ns",
        f"filtered time/pair: {r.t_fingerprint_ns:.3f} ns",
        f"speedup:            {r.speedup:.3f}",
        f"rejected:           {r.rejection_pct:.2f} % ({fs.rejected_by_fingerprint} by fingerprint, "
        f"{fs.rejected_by_length} by length, {fs.verified} verified)",
        f"construction:       {r.construction_mbps:.2f} MB/s",
        f"matches:            {r.matches_fingerprint} (naive path: {r.matches_naive})",
        f"environment:        {r.environment}",
    ]) + "\n"


def to_json_line(r) -> str:
    """report.hpp:56-83 and :96-102."""
    if isinstance(r, SweepRow):
        return json.dumps({"word_size": r.word_size, "variant": r.variant, "strategy": r.strategy,
                           "mean_pair_ns": r.mean_pair_ns})
    fs = r.filtered_stats
    return json.dumps({
        "dataset": r.dataset, "variant": _VARIANT_NAME[r.variant], "strategy": _STRATEGY_NAME[r.strategy],
        "metric": _METRIC_NAME[r.metric], "k": r.k, "word_length": r.word_length, "word_count": r.word_count,
        "letters": r.letters, "T_n_ns": r.t_naive_ns, "T_f_ns": r.t_fingerprint_ns, "speedup": r.speedup,
        "rejection_pct": r.rejection_pct, "construction_mbps": r.construction_mbps,
        "matches": r.matches_fingerprint, "matches_naive": r.matches_naive, "compared": fs.compared,
        "rejected_by_length": fs.rejected_by_length, "rejected_by_fingerprint": fs.rejected_by_fingerprint,
        "verified": fs.verified, "queries": r.query_count, "iterations": r.iterations, "seed": r.seed,
        "environment": r.environment})


# ---------------------------------------------------------------- CLI (the bench / sweep subcommands of fpbench)

def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="python -m paper_1711_08475_b200.harness")
    sub = ap.add_subparsers(dest="cmd", required=True)
    b = sub.add_parser("bench", help="run_benchmark over a word file or a synthetic English corpus")
    b.add_argument("--words", help="one word per line (default: synthetic English)")
    b.add_argument("--word-length", type=int, default=9)
    b.add_argument("--corpus-bytes", type=int, default=900_000)
    b.add_argument("--variant", choices=list(_VARIANT_NAME.values()), default="occurrence")
    b.add_argument("--strategy", choices=list(_STRATEGY_NAME.values()), default="common")
    b.add_argument("--metric", choices=list(_METRIC_NAME.values()), default="hamming")
    b.add_argument("--k", type=int, default=1)
    b.add_argument("--width", type=int, default=16)
    b.add_argument("--queries", type=int, default=1000)
    b.add_argument("--iterations", type=int, default=10)
    b.add_argument("--errors", type=int, default=1)
    b.add_argument("--seed", type=int, default=0)
    b.add_argument("--prefilter", action="store_true")
    b.add_argument("--format", choices=["text", "csv", "json"], default="text")
    s = sub.add_parser("sweep", help="emit_figure_data")
    s.add_argument("--sizes", default="5,9,13,17,21")
    s.add_argument("--corpus-bytes", type=int, default=256 * 1024)
    s.add_argument("--queries", type=int, default=200)
    s.add_argument("--format", choices=["csv", "json"], default="csv")
    a = ap.parse_args(argv)
    inv = lambda d, v: next(k for k, x in d.items() if x == v)  # noqa: E731
    if a.cmd == "bench":
        if a.words:
            with open(a.words, "rb") as f:
                words = [w.rstrip(b"\r\n") for w in f if w.strip()]
            wl = 0
        else:
            words = generate_synthetic(a.corpus_bytes, a.word_length, english_letter_frequencies(), a.seed)
            wl = a.word_length
        rep = run_benchmark(BenchConfig(dataset=a.words or "synthetic-english", words=words,
                                        variant=inv(_VARIANT_NAME, a.variant), strategy=inv(_STRATEGY_NAME, a.strategy),
                                        metric=inv(_METRIC_NAME, a.metric), k=a.k, query_count=a.queries,
                                        iterations=a.iterations, distort_max_errors=a.errors, seed=a.seed,
                                        levenshtein_length_prefilter=a.prefilter, word_length=wl, width=a.width))
        if a.format == "csv":
            print(bench_csv_header())
            print(to_csv_row(rep))
        elif a.format == "json":
            print(to_json_line(rep))
        else:
            sys.stdout.write(to_text(rep))
    else:
        rows = emit_figure_data(SweepConfig(word_sizes=[int(x) for x in a.sizes.split(",")],
                                            corpus_bytes=a.corpus_bytes, query_count=a.queries))
        if a.format == "csv":
            print(sweep_csv_header())
        for r in rows:
            print(to_csv_row(r) if a.format == "csv" else to_json_line(r))
    return 0


if __name__ == "__main__":
    sys.exit(main())
