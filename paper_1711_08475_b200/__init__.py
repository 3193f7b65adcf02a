"""B200-native fingerprint-filtered k<=1 approximate dictionary scan
(arXiv 1711.08475), behind the reference's fingerprint / matching API.

All compute runs in the CUDA library lib/libfpg.so (include/fpg.h)."""
from .fingerprints import (Batch, Fingerprint, GpuFingerprintedDictionary, LetterSet,
                           LetterStrategy, MatchCSR, Metric, QueryOptions, QueryStats, Scheme,
                           SymbolFrequencyTable, Variant, build, build_many, compute_frequencies,
                           compute_frequencies_gpu,
                           english_default_letters, english_letter_frequencies, pack_strings, render,
                           select_letters, variant_supports)

__all__ = [
    "Batch", "Fingerprint", "GpuFingerprintedDictionary", "LetterSet", "LetterStrategy",
    "MatchCSR", "Metric", "QueryOptions", "QueryStats", "Scheme", "SymbolFrequencyTable",
    "Variant", "build", "build_many", "compute_frequencies", "compute_frequencies_gpu", "english_default_letters",
    "english_letter_frequencies",
    "pack_strings", "render", "select_letters", "variant_supports",
]
