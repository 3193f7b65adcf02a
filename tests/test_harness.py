"""The GPU-backed run_benchmark / emit_figure_data harness (harness.py), the
reference's bench.hpp / report.hpp surface.  CPU tests cover the report
formats, corpora and argument checks; GPU tests the passes themselves."""
import json

import numpy as np
import pytest

from paper_1711_08475_b200 import LetterStrategy, Metric, QueryStats, Variant
from paper_1711_08475_b200.harness import (BenchConfig, BenchReport, SweepConfig, SweepRow, bench_csv_header,
                                           emit_figure_data, generate_synthetic, run_benchmark, sample_queries,
                                           sweep_csv_header, to_csv_row, to_json_line, to_text)
from paper_1711_08475_b200 import english_letter_frequencies


def test_report_headers_match_reference():
    # report.hpp:14-17 and :85-87, column for column
    assert bench_csv_header() == ("dataset,variant,strategy,metric,k,word_length,T_n_ns,T_f_ns,speedup,"
                                  "rejection_pct,construction_mbps,matches")
    assert sweep_csv_header() == "word_size,variant,strategy,mean_pair_ns"


def test_report_rows_format():
    r = BenchReport(dataset="d", variant=Variant.Count, strategy=LetterStrategy.Mixed, metric=Metric.Levenshtein,
                    k=1, word_length=9, t_naive_ns=1.23456, t_fingerprint_ns=0.5, speedup=2.46912,
                    rejection_pct=97.8412, construction_mbps=1234.5678, matches_fingerprint=42, matches_naive=42,
                    filtered_stats=QueryStats(100, 10, 80, 10, 42), word_count=100, letters="etaoinsh",
                    query_count=5, iterations=2, seed=7, environment="x")
    # fixed precision 3 for times/speedup, 2 for percentages and MB/s (report.hpp:19-27)
    assert to_csv_row(r) == "d,count,mixed,levenshtein,1,9,1.235,0.500,2.469,97.84,1234.57,42"
    assert to_csv_row(SweepRow(9, "naive", "-", 3.14159)) == "9,naive,-,3.142"
    j = json.loads(to_json_line(r))
    assert j["rejected_by_fingerprint"] == 80 and j["variant"] == "count" and j["matches_naive"] == 42
    t = to_text(r)
    assert "rejected:           97.84 % (80 by fingerprint, 10 by length, 10 verified)" in t
    assert t.startswith("dataset:            d (100 words, length 9)")


def test_synthetic_corpus_and_queries():
    w = generate_synthetic(9_000, 9, english_letter_frequencies(), seed=3)
    assert len(w) == 1000 and all(len(x) == 9 and x.isalpha() for x in w)
    assert w == generate_synthetic(9_000, 9, english_letter_frequencies(), seed=3)
    counts = np.bincount(np.frombuffer(b"".join(w), np.uint8), minlength=256)
    assert counts[ord("e")] > counts[ord("z")] * 10  # English-like
    q = sample_queries(w, 300, max_errors=1, seed=5)
    assert q == sample_queries(w, 300, max_errors=1, seed=5)
    dist = [min(sum(a != b for a, b in zip(x, y)) for y in w if len(y) == len(x)) for x in q[:50]]
    assert max(dist) <= 1 and min(dist) == 0
    with pytest.raises(ValueError):
        generate_synthetic(10, 0, english_letter_frequencies(), 1)


def test_run_benchmark_argument_checks():
    # bench.hpp:98-101 and :109-112: raised before any GPU work
    with pytest.raises(ValueError):
        run_benchmark(BenchConfig(words=[]))
    with pytest.raises(ValueError):
        run_benchmark(BenchConfig(words=[b"abc"], iterations=0))
    with pytest.raises(ValueError):
        run_benchmark(BenchConfig(words=[b"abcdefg" * 3] * 5 + [bytes(range(97, 123))],
                                  variant=Variant.Position, metric=Metric.Levenshtein))


@pytest.mark.gpu
@pytest.mark.parametrize("variant,metric", [(Variant.Occurrence, Metric.Hamming), (Variant.Count, Metric.Levenshtein),
                                            (Variant.Position, Metric.Hamming)])
def test_run_benchmark_on_gpu(oracle, variant, metric):
    """Filter-on and filter-off passes agree; the reported stats and rejection
    percentage equal the oracle's for the same words, queries and scheme."""
    from oracle.oracle import oscheme
    from paper_1711_08475_b200 import Scheme, compute_frequencies, pack_strings, select_letters

    words = generate_synthetic(60_000, 7, english_letter_frequencies(), seed=11)
    queries = sample_queries(words, 200, max_errors=1, seed=12)
    rep = run_benchmark(BenchConfig(dataset="t", words=words, variant=variant, metric=metric, query_count=200,
                                    iterations=2, queries_override=queries, word_length=7))
    assert rep.matches_naive == rep.matches_fingerprint > 0
    blob, offs = pack_strings(words)
    qb, qo = pack_strings(queries)
    cap = Scheme.letter_capacity(variant)
    sch = Scheme.make(variant, select_letters(compute_frequencies(blob), cap, LetterStrategy.Common))
    _, _, st = oracle.query_batch(blob, offs, qb, qo, oscheme(int(variant), sch.letters().symbols(), 16, 2, 3),
                                  metric, 1, True, False)
    tot = st.sum(axis=0)
    assert (rep.filtered_stats.compared, rep.filtered_stats.rejected_by_length,
            rep.filtered_stats.rejected_by_fingerprint, rep.filtered_stats.verified,
            rep.filtered_stats.matches) == tuple(int(x) for x in tot)
    pool = tot[0] - tot[1]
    assert rep.rejection_pct == pytest.approx(100.0 * tot[2] / pool)
    assert rep.t_naive_ns > 0 and rep.t_fingerprint_ns > 0 and rep.construction_mbps > 0


@pytest.mark.gpu
def test_emit_figure_data_rows():
    rows = emit_figure_data(SweepConfig(word_sizes=[5, 9], corpus_bytes=20_000, query_count=40,
                                        variants=[Variant.Occurrence, Variant.Count],
                                        strategies=[LetterStrategy.Common, LetterStrategy.Rare]))
    assert [(r.word_size, r.variant, r.strategy) for r in rows] == [
        (5, "naive", "-"), (5, "occurrence", "common"), (5, "occurrence", "rare"), (5, "count", "common"),
        (5, "count", "rare"), (9, "naive", "-"), (9, "occurrence", "common"), (9, "occurrence", "rare"),
        (9, "count", "common"), (9, "count", "rare")]
    assert all(r.mean_pair_ns > 0 for r in rows)
