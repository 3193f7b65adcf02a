// b200_ref.hpp -- the B200 dictionary as an extension of the reference library.
//
// For code that already includes the reference's own headers
// (/root/reference/proj/include/fingerprints/: corpus.hpp, reference.hpp,
// dictionary.hpp, ...): this header adds ONLY the GPU dictionary, written
// against the reference's own types -- Scheme, Fingerprint (16-bit),
// ComparisonTables, QueryOptions, QueryStats -- so one translation unit can
// hold the reference's FingerprintedDictionary, naive_scan and the GPU
// dictionary side by side.  Put the reference's include directory on the
// include path and link libfpg.so.
//
// GpuFingerprintedDictionary has the method set of FingerprintedDictionary
// (dictionary.hpp:47-125): constructor (words, scheme) (:51-56),
// words() / prints() / scheme() / tables() / size() (:58-62), query (:66-71)
// and query_into (:75-118), plus query_batch for whole batches and optional
// device sharding.  A reference caller switches by naming the type:
//     fingerprints::GpuFingerprintedDictionary dict(words, scheme);
// The fingerprints are built on the GPU (K1) and kept on the host as
// prints(); tables() is the reference's ComparisonTables of the scheme.
// Errors are the reference's: std::invalid_argument for an unsupported
// metric with the filter on (dictionary.hpp:78-79) and invalid arguments.
//
// The standalone API (fingerprints/b200.hpp, W in {16, 32, 64}, no reference
// headers) defines its own types of the same names; the two are exclusive.
#pragma once
#ifdef FPG_B200_STANDALONE_HPP
#error "fingerprints/b200_ref.hpp (reference extension) and fingerprints/b200.hpp (standalone) are exclusive"
#endif
#define FPG_B200_REF_HPP

#include <fingerprints/dictionary.hpp>  // the reference's header (its include directory on the path)

#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <string_view>
#include <vector>

#include "../fpg.h"

namespace fingerprints {

namespace b200_detail {
[[noreturn]] inline void raise(int code) {
    const std::string msg = fpg_last_error();
    if (code == FPG_EINVAL) throw std::invalid_argument(msg);
    throw std::runtime_error("fpg: " + msg);
}
inline void check(int code) {
    if (code != FPG_OK) raise(code);
}
// The reference Scheme as the C ABI's scheme (W = 16, the reference's width).
inline fpg_scheme c_scheme(const Scheme& s) {
    fpg_scheme c{};
    c.variant = static_cast<int32_t>(s.variant());
    c.width = 16;
    c.bits_per_count = static_cast<int32_t>(s.bits_per_count());
    c.bits_per_position = static_cast<int32_t>(s.bits_per_position());
    const std::size_t n = s.letters().size();
    c.nletters = static_cast<int32_t>(n);
    for (std::size_t i = 0; i < n && i < 64; ++i) c.letters[i] = s.letters().symbol(i);
    return c;
}
inline void pack(const std::vector<std::string>& v, std::string& blob, std::vector<std::uint64_t>& offs) {
    offs.assign(v.size() + 1, 0);
    blob.clear();
    for (std::size_t i = 0; i < v.size(); ++i) {
        blob += v[i];
        offs[i + 1] = blob.size();
    }
}
}  // namespace b200_detail

// Matches of a batch: query i -> word_ids[offsets[i], offsets[i+1]), ascending.
struct MatchCSR {
    std::vector<std::uint64_t> offsets;
    std::vector<std::uint32_t> word_ids;
    [[nodiscard]] std::size_t size() const { return offsets.empty() ? 0 : offsets.size() - 1; }
};

class GpuFingerprintedDictionary {
public:
    GpuFingerprintedDictionary(std::vector<std::string> words, Scheme scheme, std::vector<int> devices = {0},
                               std::uint64_t id_base = 0)
        : words_(std::move(words)), scheme_(std::move(scheme)), tables_(scheme_) {
        std::vector<std::uint64_t> offs;
        std::string blob;
        b200_detail::pack(words_, blob, offs);
        std::vector<int32_t> devs(devices.begin(), devices.end());
        const fpg_scheme s = b200_detail::c_scheme(scheme_);
        fpg_dict* d = nullptr;
        b200_detail::check(fpg_dict_create(reinterpret_cast<const std::uint8_t*>(blob.data()), offs.data(),
                                           words_.size(), &s, devs.data(), static_cast<int32_t>(devs.size()),
                                           id_base, &d));
        dict_.reset(d);
        std::vector<std::uint64_t> raw(words_.size());
        b200_detail::check(fpg_dict_prints(d, raw.data()));
        prints_.resize(raw.size());
        for (std::size_t i = 0; i < raw.size(); ++i) prints_[i].bits = static_cast<std::uint16_t>(raw[i]);
    }

    [[nodiscard]] const std::vector<std::string>& words() const { return words_; }
    [[nodiscard]] const std::vector<Fingerprint>& prints() const { return prints_; }
    [[nodiscard]] const Scheme& scheme() const { return scheme_; }
    [[nodiscard]] const ComparisonTables& tables() const { return tables_; }
    [[nodiscard]] std::size_t size() const { return words_.size(); }

    // All queries in one GPU pass; per_query (if given) receives one QueryStats per query.
    void query_batch(const std::vector<std::string>& queries, const QueryOptions& opt, MatchCSR& out,
                     std::vector<QueryStats>* per_query = nullptr) const {
        std::vector<std::uint64_t> offs;
        std::string blob;
        b200_detail::pack(queries, blob, offs);
        const fpg_query_options o{static_cast<int32_t>(opt.metric), opt.k, opt.use_filter ? 1 : 0,
                                  opt.length_prefilter ? 1 : 0, per_query ? 1 : 0, 0};
        fpg_result res{};
        b200_detail::check(fpg_query_batch(dict_.get(), reinterpret_cast<const std::uint8_t*>(blob.data()),
                                           offs.data(), queries.size(), &o, &res));
        out.offsets.assign(res.offsets, res.offsets + res.nq + 1);
        out.word_ids.assign(res.word_ids, res.word_ids + res.total);
        if (per_query) {
            per_query->resize(res.nq);
            for (std::uint64_t q = 0; q < res.nq; ++q) {
                const std::uint64_t* s = res.stats + FPG_NSTATS * q;
                (*per_query)[q] = QueryStats{s[FPG_STAT_COMPARED], s[FPG_STAT_REJECTED_BY_LENGTH],
                                             s[FPG_STAT_REJECTED_BY_FINGERPRINT], s[FPG_STAT_VERIFIED],
                                             s[FPG_STAT_MATCHES]};
            }
        }
        fpg_result_free(&res);
    }

    // dictionary.hpp:75-118: clears and refills `matches`; accumulates stats.
    void query_into(std::string_view pattern, const QueryOptions& opt, std::vector<std::size_t>& matches,
                    QueryStats* stats = nullptr) const {
        matches.clear();
        MatchCSR csr;
        std::vector<QueryStats> st;
        query_batch({std::string(pattern)}, opt, csr, stats ? &st : nullptr);
        for (std::uint64_t i = csr.offsets[0]; i < csr.offsets[1]; ++i) matches.push_back(csr.word_ids[i]);
        if (stats) *stats += st[0];
    }

    // dictionary.hpp:66-71
    [[nodiscard]] std::vector<std::size_t> query(std::string_view pattern, const QueryOptions& opt,
                                                 QueryStats* stats = nullptr) const {
        std::vector<std::size_t> m;
        query_into(pattern, opt, m, stats);
        return m;
    }

private:
    struct Deleter {
        void operator()(fpg_dict* d) const { fpg_dict_destroy(d); }
    };
    std::vector<std::string> words_;
    std::vector<Fingerprint> prints_;
    Scheme scheme_;
    ComparisonTables tables_;
    std::unique_ptr<fpg_dict, Deleter> dict_;
};

}  // namespace fingerprints
