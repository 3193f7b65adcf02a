// api_check.cpp -- compiles reference-style caller code against the B200
// headers (include/fingerprints/b200.hpp) and exercises the drop-in API.
//
//   api_check host   scheme validation / letter selection / render; no GPU
//   api_check gpu    FingerprintedDictionary::query / query_into / query_batch
//                    on cuda:0 against a brute-force scan written here
//
// The calls mirror the reference's own callers: Scheme::make + select_letters
// (bench.hpp:103-108), FingerprintedDictionary(words, scheme) and
// query(pattern, QueryOptions{metric, k, use_filter, length_prefilter})
// (dictionary_test.cpp:96, acceptance_test.cpp:283-293).
#include <fingerprints/b200.hpp>

#include <cstdio>
#include <cstdlib>
#include <random>
#include <stdexcept>
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

static int host_checks() {
    // paper schemes of "instance" (fingerprint_test.cpp:13-16 letter sets)
    const Scheme occ = Scheme::occurrence(LetterSet("etaoinshrdlcumwf"));
    CHECK(occ.field_count() == 16 && occ.width() == 16);
    const Scheme pos = Scheme::position(LetterSet("etaoin"), 3);
    CHECK(pos.field_count() == 6 && pos.field_shift(0) == 13 && pos.field_shift(5) == 0);
    const Scheme cnt = Scheme::count(LetterSet("etaoinsh"), 2);
    CHECK(cnt.field_count() == 8 && cnt.field_width(3) == 2 && cnt.field_shift(7) == 0);
    CHECK(render(Fingerprint{0x5a5a}, cnt) == "01 01 10 10 01 01 10 10");
    bool threw = false;
    try {
        (void)Scheme::occurrence(LetterSet("etaoin"));  // 6 letters for a 16-bit occurrence scheme
    } catch (const std::invalid_argument&) {
        threw = true;
    }
    CHECK(threw);
    threw = false;
    try {
        (void)LetterSet("aa");
    } catch (const std::invalid_argument&) {
        threw = true;
    }
    CHECK(threw);
    CHECK(!variant_supports(Variant::Position, Metric::Levenshtein));
    CHECK(Scheme::letter_capacity(Variant::Position, 2, 3, 64) == 22);
    const auto freq = compute_frequencies(std::vector<std::string>{"banana", "bandana", "cab"});
    const LetterSet common = select_letters(freq, 2, LetterStrategy::Common);
    CHECK(common.symbols() == "an");
    // ComparisonTables / fingerprint_distance / can_reject generalised to W
    // (fingerprint.hpp:171-214, :287-301) vs a field-by-field count
    // (reference.hpp:62-84 restated with 16 -> W)
    std::mt19937_64 rng(3);
    const std::string az = "abcdefghijklmnopqrstuvwxyz0123456789ABCDEFGHIJKLMNOPQRSTUVWXYZ!?";
    for (int width : {16, 32, 64})
        for (Variant v : {Variant::Occurrence, Variant::OccurrenceHalved, Variant::Count, Variant::Position}) {
            const unsigned b = v == Variant::Count && width == 64 ? 4 : 2;
            const std::size_t cap = Scheme::letter_capacity(v, b, 3, width);
            const Scheme s = Scheme::make(v, LetterSet(az.substr(0, cap)), b, 3, width);
            const ComparisonTables t(s);
            CHECK(t.width() == width && t.has_group_table() == (v == Variant::Count || v == Variant::Position));
            const std::uint64_t wmask = width == 64 ? ~0ull : (1ull << width) - 1;
            for (int i = 0; i < 4000; ++i) {
                const Fingerprint x{rng() & wmask}, y{(rng() & rng()) & wmask};
                const std::uint64_t d = x.bits ^ y.bits;
                int fd = 0;
                if (t.has_group_table()) {
                    for (std::size_t f = 0; f < s.field_count(); ++f)
                        fd += ((d >> s.field_shift(f)) & ((1ull << s.field_width(f)) - 1)) != 0;
                } else {
                    for (int bit = 0; bit < width; ++bit) fd += (d >> bit) & 1;
                }
                CHECK(fingerprint_distance(x, y, s, t) == fd);
                CHECK(lower_bound_errors(fd, t) == (fd + 1) / 2);
                for (int k = 0; k <= 3; ++k) CHECK(can_reject(x, y, k, s, t) == ((fd + 1) / 2 > k));
            }
        }
    std::puts("api_check host: ok");
    return 0;
}

static bool hamming_le(const std::string& a, const std::string& b, int k) {
    if (a.size() != b.size()) return false;
    int d = 0;
    for (size_t i = 0; i < a.size(); ++i) d += a[i] != b[i];
    return d <= k;
}

static bool lev_le1(const std::string& a, const std::string& b) {
    if (a == b) return true;
    const std::string& s = a.size() >= b.size() ? a : b;  // longer
    const std::string& t = a.size() >= b.size() ? b : a;
    if (s.size() == t.size()) return hamming_le(s, t, 1);
    if (s.size() != t.size() + 1) return false;
    for (size_t i = 0; i < s.size(); ++i)
        if (s.substr(0, i) + s.substr(i + 1) == t) return true;
    return false;
}

static int gpu_checks() {
    std::mt19937_64 rng(7);
    std::vector<std::string> words;
    for (int i = 0; i < 3000; ++i) {
        std::string w(4 + rng() % 5, 'a');
        for (char& c : w) c = static_cast<char>('a' + rng() % 10);
        words.push_back(w);
    }
    std::vector<std::string> queries;
    for (int i = 0; i < 40; ++i) {
        std::string q = words[rng() % words.size()];
        q[rng() % q.size()] = static_cast<char>('a' + rng() % 10);
        queries.push_back(q);
    }
    const Scheme scheme = Scheme::make(Variant::Count, select_letters(compute_frequencies(words), 8,
                                                                    LetterStrategy::Common));
    FingerprintedDictionary dict(words, scheme);
    CHECK(dict.size() == words.size());
    for (Metric m : {Metric::Hamming, Metric::Levenshtein}) {
        const QueryOptions opt{m, 1, true, false};
        MatchCSR csr;
        std::vector<QueryStats> per;
        dict.query_batch(queries, opt, csr, &per);
        for (size_t q = 0; q < queries.size(); ++q) {
            std::vector<std::size_t> want;
            for (size_t w = 0; w < words.size(); ++w)
                if (m == Metric::Hamming ? hamming_le(words[w], queries[q], 1) : lev_le1(words[w], queries[q]))
                    want.push_back(w);
            QueryStats st;
            const std::vector<std::size_t> got = dict.query(queries[q], opt, &st);
            CHECK(got == want);
            CHECK(csr.offsets[q + 1] - csr.offsets[q] == want.size());
            for (size_t i = 0; i < want.size(); ++i) CHECK(csr.word_ids[csr.offsets[q] + i] == want[i]);
            CHECK(st.compared == words.size() && st.matches == want.size());
            CHECK(st.rejected_by_length + st.rejected_by_fingerprint + st.verified == st.compared);
            CHECK(per[q].verified == st.verified && per[q].rejected_by_length == st.rejected_by_length);
            // every match survives the host pair test with the dictionary's tables()
            const Fingerprint qp = build(queries[q], scheme);
            const std::vector<Fingerprint> prints = dict.prints();
            for (std::size_t id : got) CHECK(!can_reject(qp, prints[id], 1, scheme, dict.tables()));
        }
    }
    // the same dictionary split from its newline text on the GPU
    std::string text;
    for (const auto& w : words) text += w + "\n";
    const FingerprintedDictionary from_text = FingerprintedDictionary::from_text(text, scheme);
    CHECK(from_text.size() == words.size());
    CHECK(from_text.prints() == dict.prints());
    const auto freq_gpu = compute_frequencies_gpu(text);
    CHECK(freq_gpu.counts[static_cast<unsigned char>('\n')] == words.size());
    bool threw = false;
    try {
        const Scheme p = Scheme::position(select_letters(compute_frequencies(words), 6, LetterStrategy::Common));
        FingerprintedDictionary d2(words, p);
        (void)d2.query(queries[0], QueryOptions{Metric::Levenshtein, 1, true, false});
    } catch (const std::invalid_argument&) {
        threw = true;
    }
    CHECK(threw);
    std::puts("api_check gpu: ok");
    return 0;
}

int main(int argc, char** argv) {
    const std::string mode = argc > 1 ? argv[1] : "host";
    return mode == "gpu" ? gpu_checks() : host_checks();
}
