// api_check_ref.cpp -- the GPU dictionary as an extension of the reference
// library: ONE translation unit holds the reference's corpus generator
// (corpus.hpp), FingerprintedDictionary (dictionary.hpp), naive_scan
// (reference.hpp) and fingerprints::GpuFingerprintedDictionary
// (include/fingerprints/b200_ref.hpp), over the reference's own Scheme,
// Fingerprint, ComparisonTables, QueryOptions and QueryStats.
//
//   api_check_ref host   reference-side checks only (no GPU): the types the
//                        GPU dictionary exposes are the reference's, and
//                        tables()/can_reject agree with reference.hpp's
//                        field-by-field distance
//   api_check_ref gpu    for every variant x metric the reference filters:
//                        GPU prints() == reference prints(), GPU query() ==
//                        reference query() == naive_scan, QueryStats equal,
//                        and every GPU match passes can_reject(..) == false
//                        with the GPU dictionary's tables()
//
// Built by __graft_entry__.build() when the reference tree exists
// (tests/cpp/_bin/api_check_ref, it travels to the GPU box) and run by
// tests/test_gpu_parity.py::test_cpp_reference_extension.
#include <fingerprints/corpus.hpp>
#include <fingerprints/dictionary.hpp>
#include <fingerprints/reference.hpp>

#include <fingerprints/b200_ref.hpp>

#include <cstdio>
#include <cstdlib>
#include <random>
#include <string>
#include <vector>

using namespace fingerprints;

#define CHECK(c)                                                              \
    do {                                                                      \
        if (!(c)) {                                                           \
            std::fprintf(stderr, "FAIL %s:%d: %s\n", __FILE__, __LINE__, #c); \
            std::exit(1);                                                     \
        }                                                                     \
    } while (0)

namespace {

std::vector<std::string> corpus() {
    // fixed-length English-frequency words (corpus.hpp:44-70), lengths 3..8
    std::vector<std::string> words;
    for (std::size_t len = 3; len <= 8; ++len) {
        auto part = generate_synthetic(2500 * len, len, english_letter_frequencies(), 11 + len);
        words.insert(words.end(), part.begin(), part.end());
    }
    return words;
}

std::vector<Scheme> schemes(const std::vector<std::string>& words) {
    const SymbolFrequencyTable freq = compute_frequencies(words);
    std::vector<Scheme> out;
    for (Variant v : {Variant::Occurrence, Variant::OccurrenceHalved, Variant::Count, Variant::Position}) {
        const std::size_t cap = Scheme::letter_capacity(v, 2, 3);
        out.push_back(Scheme::make(v, select_letters(freq, cap, LetterStrategy::Common), 2, 3));
    }
    return out;
}

int host_checks() {
    const auto words = corpus();
    std::mt19937_64 rng(7);
    for (const Scheme& s : schemes(words)) {
        const ComparisonTables t(s);
        for (int i = 0; i < 20000; ++i) {
            const Fingerprint a{static_cast<std::uint16_t>(rng())}, b{static_cast<std::uint16_t>(rng())};
            const int fd = fingerprint_distance_reference(a, b, s);
            CHECK(fingerprint_distance(a, b, s, t) == fd);
            for (int k = 0; k <= 3; ++k) CHECK(can_reject(a, b, k, s, t) == ((fd + 1) / 2 > k));
        }
    }
    std::puts("api_check_ref host: ok");
    return 0;
}

int gpu_checks() {
    const auto words = corpus();
    const auto queries = sample_queries(words, 300, {2, 0.5}, 5);
    std::size_t total_matches = 0;
    for (const Scheme& s : schemes(words)) {
        const FingerprintedDictionary ref(words, s);
        const GpuFingerprintedDictionary gpu(words, s);
        CHECK(gpu.size() == ref.size());
        CHECK(gpu.prints().size() == ref.prints().size());
        for (std::size_t i = 0; i < ref.prints().size(); ++i) CHECK(gpu.prints()[i] == ref.prints()[i]);
        for (Metric m : {Metric::Hamming, Metric::Levenshtein}) {
            if (!s.supports(m)) {
                bool threw = false;
                try {
                    (void)gpu.query("abc", QueryOptions{m, 1, true, false});
                } catch (const std::invalid_argument&) {
                    threw = true;
                }
                CHECK(threw);  // dictionary.hpp:78-79
                continue;
            }
            for (int k : {0, 1}) {
                // the GPU length-buckets; the reference's stats match it with the prefilter on
                const QueryOptions opt{m, k, true, true};
                std::vector<std::size_t> got;
                for (const auto& q : queries) {
                    QueryStats gs, rs;
                    gpu.query_into(q, opt, got, &gs);
                    const auto want = ref.query(q, opt, &rs);
                    CHECK(got == want);
                    CHECK(got == naive_scan(words, q, k, m));
                    CHECK(gs.compared == rs.compared && gs.rejected_by_length == rs.rejected_by_length &&
                          gs.rejected_by_fingerprint == rs.rejected_by_fingerprint && gs.verified == rs.verified &&
                          gs.matches == rs.matches);
                    const Fingerprint qp = build(q, s);
                    for (std::size_t id : got) CHECK(!can_reject(qp, gpu.prints()[id], k, s, gpu.tables()));
                    total_matches += got.size();
                }
                MatchCSR csr;
                gpu.query_batch(queries, opt, csr);
                CHECK(csr.size() == queries.size());
                for (std::size_t i = 0; i < queries.size(); ++i) {
                    const auto want = ref.query(queries[i], opt);
                    CHECK(csr.offsets[i + 1] - csr.offsets[i] == want.size());
                    for (std::size_t j = 0; j < want.size(); ++j) CHECK(csr.word_ids[csr.offsets[i] + j] == want[j]);
                }
            }
        }
    }
    CHECK(total_matches > 0);
    std::printf("api_check_ref gpu: ok (%zu matches)\n", total_matches);
    return 0;
}

}  // namespace

int main(int argc, char** argv) {
    const std::string mode = argc > 1 ? argv[1] : "host";
    if (mode == "host") return host_checks();
    if (mode == "gpu") return gpu_checks();
    std::fprintf(stderr, "usage: api_check_ref host|gpu\n");
    return 2;
}
