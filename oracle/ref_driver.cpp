// ref_driver.cpp -- extern "C" shim over the UNMODIFIED reference headers.
//
// TEST INFRASTRUCTURE ONLY.  Compiled by oracle/Makefile against
// /root/reference/proj/include (header-only C++20) into oracle/_ref/libfpref.so.
// It adds no algorithm of its own: every entry point forwards to the
// reference's public API (fingerprint.hpp build/render/can_reject,
// edit_distance.hpp verifiers, dictionary.hpp FingerprintedDictionary::query_into,
// reference.hpp naive_scan, letter_model.hpp select_letters).  Used to pin the
// C restatement (fp_oracle.c) at W=16 and as the CPU baseline ("kind":
// "reference") in bench.py.  No reference source is copied into this repo.
#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "fingerprints/dictionary.hpp"
#include "fingerprints/edit_distance.hpp"
#include "fingerprints/fingerprint.hpp"
#include "fingerprints/letter_model.hpp"
#include "fingerprints/reference.hpp"

using namespace fingerprints;

namespace {

Scheme make_scheme(int variant, const unsigned char* letters, int nletters, int b, int p) {
    LetterSet ls(std::string_view(reinterpret_cast<const char*>(letters), (size_t)nletters));
    return Scheme::make(static_cast<Variant>(variant), ls, (unsigned)b, (unsigned)p);
}

std::vector<std::string> split(const unsigned char* blob, const uint64_t* offs, uint64_t n) {
    std::vector<std::string> v;
    v.reserve(n);
    for (uint64_t i = 0; i < n; ++i)
        v.emplace_back(reinterpret_cast<const char*>(blob + offs[i]), offs[i + 1] - offs[i]);
    return v;
}

struct Handle {
    FingerprintedDictionary dict;
    Handle(std::vector<std::string> w, Scheme s) : dict(std::move(w), std::move(s)) {}
};

}  // namespace

extern "C" {

// Scheme::make + LetterSet ctor validation. 0 ok, -1 invalid_argument.
int fpr_scheme_check(int variant, const unsigned char* letters, int nletters, int b, int p) {
    try {
        make_scheme(variant, letters, nletters, b, p);
        return 0;
    } catch (const std::invalid_argument&) {
        return -1;
    }
}

int fpr_letter_capacity(int variant, int b, int p) {
    try {
        return (int)Scheme::letter_capacity(static_cast<Variant>(variant), (unsigned)b, (unsigned)p);
    } catch (const std::invalid_argument&) {
        return -1;
    }
}

int fpr_select_letters(const unsigned char* bytes, uint64_t nbytes, int count, int strategy,
                       unsigned char* out) {
    try {
        auto freq = compute_frequencies(std::string_view(reinterpret_cast<const char*>(bytes), nbytes));
        LetterSet ls = select_letters(freq, (size_t)count, static_cast<LetterStrategy>(strategy));
        std::memcpy(out, ls.symbols().data(), ls.size());
        return (int)ls.size();
    } catch (const std::invalid_argument&) {
        return -1;
    }
}

int fpr_build_many(const unsigned char* blob, const uint64_t* offs, uint64_t n, int variant,
                   const unsigned char* letters, int nletters, int b, int p, uint16_t* out) {
    try {
        Scheme s = make_scheme(variant, letters, nletters, b, p);
        for (uint64_t i = 0; i < n; ++i)
            out[i] = build(std::string_view(reinterpret_cast<const char*>(blob + offs[i]),
                                            offs[i + 1] - offs[i]),
                           s)
                         .bits;
        return 0;
    } catch (const std::invalid_argument&) {
        return -1;
    }
}

// Table distance (ComparisonTables::distance) for each xor value in [0, 2^16).
int fpr_distance_table(int variant, const unsigned char* letters, int nletters, int b, int p,
                       uint8_t* out65536) {
    try {
        Scheme s = make_scheme(variant, letters, nletters, b, p);
        ComparisonTables t(s);
        for (uint32_t x = 0; x < 65536; ++x)
            out65536[x] = (uint8_t)t.distance(Fingerprint{(uint16_t)x}, Fingerprint{0});
        return 0;
    } catch (const std::invalid_argument&) {
        return -1;
    }
}

int fpr_render(uint16_t f, int variant, const unsigned char* letters, int nletters, int b, int p,
               char* out) {
    try {
        Scheme s = make_scheme(variant, letters, nletters, b, p);
        std::string r = render(Fingerprint{f}, s);
        std::memcpy(out, r.c_str(), r.size() + 1);
        return 0;
    } catch (const std::invalid_argument&) {
        return -1;
    }
}

int fpr_hamming_bounded(const unsigned char* a, size_t na, const unsigned char* b, size_t nb, int k) {
    try {
        auto r = hamming_bounded(std::string_view((const char*)a, na), std::string_view((const char*)b, nb), k);
        return r ? *r : -1;
    } catch (const std::invalid_argument&) {
        return -2;
    }
}

int fpr_levenshtein_bounded(const unsigned char* a, size_t na, const unsigned char* b, size_t nb,
                            int k) {
    auto r = levenshtein_bounded(std::string_view((const char*)a, na), std::string_view((const char*)b, nb), k);
    return r ? *r : -1;
}

int fpr_levenshtein_full(const unsigned char* a, size_t na, const unsigned char* b, size_t nb) {
    return levenshtein_full(std::string_view((const char*)a, na), std::string_view((const char*)b, nb));
}

// Builds a FingerprintedDictionary (the reference ctor: fingerprints + tables).
void* fpr_dict_create(const unsigned char* blob, const uint64_t* offs, uint64_t n, int variant,
                      const unsigned char* letters, int nletters, int b, int p) {
    try {
        return new Handle(split(blob, offs, n), make_scheme(variant, letters, nletters, b, p));
    } catch (const std::invalid_argument&) {
        return nullptr;
    }
}

void fpr_dict_destroy(void* h) { delete static_cast<Handle*>(h); }

// query_into for every query, queries partitioned over nthreads std::threads
// (concurrent const queries are safe, README.md:124-125).  CSR outputs as in
// fp_oracle.h.  Returns -1 on invalid_argument (unsupported metric).
int fpr_query_batch(void* h, const unsigned char* qblob, const uint64_t* qoffs, uint64_t nq,
                    int metric, int k, int use_filter, int length_prefilter, int nthreads,
                    uint64_t* offsets, uint64_t* stats, uint32_t** ids, uint64_t* total) {
    const auto& dict = static_cast<Handle*>(h)->dict;
    QueryOptions opt{static_cast<Metric>(metric), k, use_filter != 0, length_prefilter != 0};
    if (opt.use_filter && !dict.scheme().supports(opt.metric))
        return -1;
    if (nthreads < 1) nthreads = 1;
    if ((uint64_t)nthreads > nq) nthreads = nq ? (int)nq : 1;
    std::vector<std::vector<uint32_t>> out((size_t)nthreads);
    std::vector<uint64_t> counts(nq);
    auto work = [&](int t) {
        const uint64_t q0 = nq * (uint64_t)t / (uint64_t)nthreads;
        const uint64_t q1 = nq * (uint64_t)(t + 1) / (uint64_t)nthreads;
        std::vector<std::size_t> matches;
        for (uint64_t q = q0; q < q1; ++q) {
            QueryStats st;
            dict.query_into(std::string_view((const char*)qblob + qoffs[q], qoffs[q + 1] - qoffs[q]),
                            opt, matches, &st);
            counts[q] = matches.size();
            for (auto m : matches) out[(size_t)t].push_back((uint32_t)m);
            if (stats) {
                uint64_t* s = stats + 5 * q;
                s[0] = st.compared; s[1] = st.rejected_by_length; s[2] = st.rejected_by_fingerprint;
                s[3] = st.verified; s[4] = st.matches;
            }
        }
    };
    std::vector<std::thread> th;
    for (int t = 1; t < nthreads; ++t) th.emplace_back(work, t);
    work(0);
    for (auto& x : th) x.join();
    uint64_t tot = 0;
    offsets[0] = 0;
    for (uint64_t q = 0; q < nq; ++q) { tot += counts[q]; offsets[q + 1] = tot; }
    uint32_t* res = static_cast<uint32_t*>(std::malloc(sizeof(uint32_t) * (tot ? tot : 1)));
    uint64_t pos = 0;
    for (auto& v : out) {
        if (!v.empty()) std::memcpy(res + pos, v.data(), v.size() * sizeof(uint32_t));
        pos += v.size();
    }
    *ids = res;
    *total = tot;
    return 0;
}

// naive_scan (reference.hpp:45-59) for one query.
int fpr_naive_scan(const unsigned char* blob, const uint64_t* offs, uint64_t n,
                   const unsigned char* q, size_t nqlen, int metric, int k, uint32_t* out,
                   uint64_t cap, uint64_t* count) {
    auto words = split(blob, offs, n);
    auto m = naive_scan(words, std::string_view((const char*)q, nqlen), k, static_cast<Metric>(metric));
    *count = m.size();
    for (size_t i = 0; i < m.size() && i < cap; ++i) out[i] = (uint32_t)m[i];
    return 0;
}

void fpr_free(void* p) { std::free(p); }

}  // extern "C"
