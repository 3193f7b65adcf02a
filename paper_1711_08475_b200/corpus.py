"""Seeded synthetic inputs for the five BASELINE configs (BASELINE.json:7-11).

Generation runs in libfpcorpus.so (csrc/corpus/fpcorpus.c): counter-based
streams, so word i of a dictionary does not depend on N or on thread count
and a larger dictionary extends a smaller one.  Resolutions of the configs'
conflicts with the reference live in CELLS below.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from ._lib import host_threads, load_corpus
from .fingerprints import (LetterStrategy, Metric, Scheme, Variant, compute_frequencies,
                           select_letters)


@dataclass(frozen=True)
class Config:
    cfg: int
    seed: int
    n_words: int
    n_queries: int
    description: str


CONFIGS = {
    1: Config(1, 1, 100_000, 1_000, "a-z uniform, L~U[4,16]; 50% one-substitution / 50% random"),
    2: Config(2, 2, 1_000_000, 10_000, "a-z uniform, L~U[4,20]; 1/3 exact / 1/3 one edit / 1/3 random"),
    3: Config(3, 3, 2_000_000, 50_000, "English categorical, L=2+Geom trunc [2,24] mean 8; 50% one edit / 50% random"),
    4: Config(4, 4, 8_000_000, 100_000, "URL-like, 46-symbol alphabet, L in [20,100] mean ~45; 50% one edit / 50% random"),
    5: Config(5, 5, 64_000_000, 1_000_000, "a-z uniform, L~U[4,16]; 50% one edit / 50% random; sharded"),
}

# Scheme cells per config: (variant, width, b, p, metric).  Unsound or
# infeasible cells are dropped: halved/position never
# filter Levenshtein (fingerprint.hpp:36-38); widths whose letter capacity
# exceeds the alphabet are infeasible (letter_model.hpp:106-109).
H, L = Metric.Hamming, Metric.Levenshtein
V = Variant
CELLS = {
    1: [(V.Occurrence, 16, 2, 3, H)],
    2: [(V.Count, 16, 2, 3, L)],
    3: [(V.Occurrence, 16, 2, 3, H), (V.Occurrence, 16, 2, 3, L),
        (V.OccurrenceHalved, 16, 2, 3, H), (V.OccurrenceHalved, 32, 2, 3, H)],
    4: [(V.Position, 64, 2, 3, H), (V.Count, 64, 4, 3, L)],
    5: [(V.Occurrence, 16, 2, 3, H), (V.Occurrence, 16, 2, 3, L),
        (V.OccurrenceHalved, 16, 2, 3, H), (V.OccurrenceHalved, 32, 2, 3, H),
        (V.Count, 16, 2, 3, H), (V.Count, 16, 2, 3, L),
        (V.Count, 32, 2, 3, H), (V.Count, 32, 2, 3, L),
        (V.Position, 16, 2, 3, H), (V.Position, 32, 2, 3, H), (V.Position, 64, 2, 3, H)],
}


def generate_dictionary(cfg: int, n: int | None = None, seed: int | None = None,
                        threads: int | None = None, first: int = 0) -> tuple[np.ndarray, np.ndarray]:
    """(blob uint8, offsets uint64[n+1]) of words [first, first+n) of the
    config's dictionary stream (first > 0: a shard of a larger dictionary)."""
    c = CONFIGS[cfg]
    n = c.n_words if n is None else n
    seed = c.seed if seed is None else seed
    lib = load_corpus()
    th = threads or min(host_threads(), 32)
    offsets = np.zeros(n + 1, dtype=np.uint64)
    total = lib.fpc_dict_lengths_at(cfg, seed, first, n, offsets.ctypes.data, th)
    if total < 0:
        raise ValueError(f"unknown config {cfg}")
    blob = np.zeros(max(total, 1), dtype=np.uint8)
    lib.fpc_dict_fill_at(cfg, seed, first, n, offsets.ctypes.data, blob.ctypes.data, th)
    return blob[:total], offsets


def generate_queries(cfg: int, dblob: np.ndarray, doffs: np.ndarray, nq: int | None = None,
                     seed: int | None = None, n_base: int | None = None) -> tuple[np.ndarray, np.ndarray]:
    c = CONFIGS[cfg]
    nq = c.n_queries if nq is None else nq
    seed = c.seed if seed is None else seed
    n_base = len(doffs) - 1 if n_base is None else n_base
    lib = load_corpus()
    cap = max(nq * lib.fpc_max_len(cfg), 1)
    qblob = np.zeros(cap, dtype=np.uint8)
    qoffs = np.zeros(nq + 1, dtype=np.uint64)
    used = lib.fpc_queries(cfg, seed, dblob.ctypes.data, doffs.ctypes.data, n_base, nq,
                           qblob.ctypes.data, cap, qoffs.ctypes.data)
    if used < 0:
        raise ValueError(f"query generation failed ({used})")
    return qblob[:used].copy(), qoffs


def make_scheme(blob: np.ndarray, variant: Variant, width: int, b: int = 2, p: int = 3,
                strategy: LetterStrategy = LetterStrategy.Common) -> Scheme:
    """Letters chosen over the WHOLE dictionary, then the scheme."""
    cap = Scheme.letter_capacity(variant, b, p, width)
    letters = select_letters(compute_frequencies(blob), cap, strategy)
    return Scheme.make(variant, letters, b, p, width)


def subsample(qblob: np.ndarray, qoffs: np.ndarray, step: int) -> tuple[np.ndarray, np.ndarray, np.ndarray]:
    """Every `step`-th query (deterministic subsample)."""
    idx = np.arange(0, len(qoffs) - 1, step)
    parts = [qblob[int(qoffs[i]):int(qoffs[i + 1])] for i in idx]
    offs = np.zeros(len(idx) + 1, dtype=np.uint64)
    offs[1:] = np.cumsum([len(x) for x in parts])
    blob = np.concatenate(parts) if parts else np.zeros(0, np.uint8)
    return blob, offs, idx
