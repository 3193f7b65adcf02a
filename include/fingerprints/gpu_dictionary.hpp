// gpu_dictionary.hpp -- the B200 dictionary behind the reference's matching API.
//
// GpuFingerprintedDictionary has the method set of the reference's
// FingerprintedDictionary (dictionary.hpp:47-125): the constructor
// (words, scheme) (:51-56), words()/prints()/scheme()/size() (:58-62),
// query (:66-71) and query_into (:75-118) with QueryOptions (:36-44) and
// accumulating QueryStats (:19-34), plus query_batch for whole batches.  All
// work runs in libfpg.so (include/fpg.h); the words may be sharded over
// several GPUs.  Errors are rethrown as the reference throws them:
// std::invalid_argument for invalid schemes and unsupported metrics.
#pragma once

#include <cstdint>
#include <memory>
#include <string>
#include <string_view>
#include <vector>

#include "gpu_scheme.hpp"

namespace fingerprints {

struct QueryStats {
    std::uint64_t compared = 0;
    std::uint64_t rejected_by_length = 0;
    std::uint64_t rejected_by_fingerprint = 0;
    std::uint64_t verified = 0;
    std::uint64_t matches = 0;

    QueryStats& operator+=(const QueryStats& o) {
        compared += o.compared;
        rejected_by_length += o.rejected_by_length;
        rejected_by_fingerprint += o.rejected_by_fingerprint;
        verified += o.verified;
        matches += o.matches;
        return *this;
    }
};

// Field order kept: callers aggregate-initialise it positionally.
struct QueryOptions {
    Metric metric = Metric::Hamming;
    int k = 1;
    bool use_filter = true;
    bool length_prefilter = false;
};

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
        : words_(std::move(words)), scheme_(std::move(scheme)), tables_(scheme_), n_(words_.size()) {
        std::vector<std::uint64_t> offs(words_.size() + 1, 0);
        std::string blob;
        for (std::size_t i = 0; i < words_.size(); ++i) {
            blob += words_[i];
            offs[i + 1] = blob.size();
        }
        std::vector<int32_t> devs(devices.begin(), devices.end());
        const fpg_scheme s = scheme_.c_struct();
        fpg_dict* d = nullptr;
        detail::check(fpg_dict_create(reinterpret_cast<const std::uint8_t*>(blob.data()), offs.data(), words_.size(),
                                      &s, devs.data(), static_cast<int32_t>(devs.size()), id_base, &d));
        dict_.reset(d);
    }

    // Newline-separated word text (read_word_lines, corpus.hpp:116-125) split
    // into words on the GPU(s); words() stays empty.
    static GpuFingerprintedDictionary from_text(std::string_view text, Scheme scheme, std::vector<int> devices = {0},
                                                std::uint64_t id_base = 0) {
        GpuFingerprintedDictionary d(std::move(scheme));
        std::vector<int32_t> devs(devices.begin(), devices.end());
        const fpg_scheme s = d.scheme_.c_struct();
        fpg_dict* h = nullptr;
        detail::check(fpg_dict_create_from_text(reinterpret_cast<const std::uint8_t*>(text.data()), text.size(), &s,
                                                devs.data(), static_cast<int32_t>(devs.size()), id_base, &h));
        d.dict_.reset(h);
        std::uint64_t n = 0;
        detail::check(fpg_dict_size(h, &n));
        d.n_ = n;
        return d;
    }

    [[nodiscard]] const std::vector<std::string>& words() const { return words_; }
    [[nodiscard]] const Scheme& scheme() const { return scheme_; }
    /// dictionary.hpp:61: the host-side pair tables of the scheme (the GPU
    /// scan applies the same F_D > 2k test bit-sliced).
    [[nodiscard]] const ComparisonTables& tables() const { return tables_; }
    [[nodiscard]] std::size_t size() const { return n_; }
    [[nodiscard]] std::vector<Fingerprint> prints() const {
        std::vector<std::uint64_t> raw(n_);
        detail::check(fpg_dict_prints(dict_.get(), raw.data()));
        std::vector<Fingerprint> out(raw.size());
        for (std::size_t i = 0; i < raw.size(); ++i) out[i].bits = raw[i];
        return out;
    }

    // All queries in one GPU pass; per_query (if given) receives one QueryStats per query.
    void query_batch(const std::vector<std::string>& queries, const QueryOptions& opt, MatchCSR& out,
                     std::vector<QueryStats>* per_query = nullptr) const {
        std::vector<std::uint64_t> offs(queries.size() + 1, 0);
        std::string blob;
        for (std::size_t i = 0; i < queries.size(); ++i) {
            blob += queries[i];
            offs[i + 1] = blob.size();
        }
        const fpg_query_options o{static_cast<int32_t>(opt.metric), opt.k, opt.use_filter ? 1 : 0,
                                  opt.length_prefilter ? 1 : 0, per_query ? 1 : 0, 0};
        fpg_result res{};
        detail::check(fpg_query_batch(dict_.get(), reinterpret_cast<const std::uint8_t*>(blob.data()), offs.data(),
                                      queries.size(), &o, &res));
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

    // Clears and refills `matches` with input-order ids; accumulates stats.
    void query_into(std::string_view pattern, const QueryOptions& opt, std::vector<std::size_t>& matches,
                    QueryStats* stats = nullptr) const {
        matches.clear();
        MatchCSR csr;
        std::vector<QueryStats> st;
        query_batch({std::string(pattern)}, opt, csr, stats ? &st : nullptr);
        for (std::uint64_t i = csr.offsets[0]; i < csr.offsets[1]; ++i) matches.push_back(csr.word_ids[i]);
        if (stats) *stats += st[0];
    }

    [[nodiscard]] std::vector<std::size_t> query(std::string_view pattern, const QueryOptions& opt,
                                                 QueryStats* stats = nullptr) const {
        std::vector<std::size_t> m;
        query_into(pattern, opt, m, stats);
        return m;
    }

private:
    explicit GpuFingerprintedDictionary(Scheme scheme) : scheme_(std::move(scheme)), tables_(scheme_) {}
    struct Deleter {
        void operator()(fpg_dict* d) const { fpg_dict_destroy(d); }
    };
    std::vector<std::string> words_;
    Scheme scheme_;
    ComparisonTables tables_;
    std::uint64_t n_ = 0;
    std::unique_ptr<fpg_dict, Deleter> dict_;
};

}  // namespace fingerprints
