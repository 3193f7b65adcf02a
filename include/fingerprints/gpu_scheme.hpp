// gpu_scheme.hpp -- fingerprint schemes of the B200 build (host side).
//
// Mirrors the reference's fingerprint.hpp interface: Variant / Metric (:14-15),
// variant_supports (:36-38), Fingerprint (:41-44), Scheme (:57-162) and
// render (:305-317), ComparisonTables / fingerprint_distance /
// lower_bound_errors / can_reject (:171-214, :287-301), plus the fingerprint
// width W in {16, 32, 64} that the reference fixes at 16 (:31).  build()
// runs on the GPU (K1 of libfpg.so); the pair test runs on the host here for
// callers that test single pairs (the GPU scan evaluates the same F_D > 2k
// rule bit-sliced, fpg_slice.cuh).
//
// This is the standalone API (no reference headers needed; Fingerprint::bits
// is 64-bit so W = 32 / 64 fit).  Code that also includes the reference's own
// headers uses fingerprints/b200_ref.hpp instead, which adds only the GPU
// dictionary on top of the reference's types.
#pragma once
#ifdef FPG_B200_REF_HPP
#error "fingerprints/b200.hpp (standalone) and fingerprints/b200_ref.hpp (reference extension) are exclusive"
#endif
#define FPG_B200_STANDALONE_HPP

#include <array>
#include <bit>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <string_view>
#include <vector>

#include "../fpg.h"
#include "gpu_letters.hpp"

namespace fingerprints {

enum class Variant { Occurrence = FPG_OCCURRENCE, OccurrenceHalved = FPG_OCCURRENCE_HALVED, Count = FPG_COUNT,
                     Position = FPG_POSITION };
enum class Metric { Hamming = FPG_HAMMING, Levenshtein = FPG_LEVENSHTEIN };

inline std::string_view to_string(Variant v) {
    switch (v) {
        case Variant::Occurrence: return "occurrence";
        case Variant::OccurrenceHalved: return "occurrence-halved";
        case Variant::Count: return "count";
        case Variant::Position: return "position";
    }
    return "?";
}
inline std::string_view to_string(Metric m) { return m == Metric::Hamming ? "hamming" : "levenshtein"; }

inline constexpr bool variant_supports(Variant v, Metric m) {
    return m == Metric::Hamming || v == Variant::Occurrence || v == Variant::Count;
}

struct Fingerprint {
    std::uint64_t bits = 0;
    friend bool operator==(Fingerprint, Fingerprint) = default;
};

namespace detail {
[[noreturn]] inline void raise(int code) {
    const std::string msg = fpg_last_error();
    if (code == FPG_EINVAL) throw std::invalid_argument(msg);
    throw std::runtime_error("fpg: " + msg);
}
inline void check(int code) {
    if (code != FPG_OK) raise(code);
}
}  // namespace detail

class Scheme {
public:
    static Scheme occurrence(LetterSet l, int width = 16) { return Scheme(Variant::Occurrence, std::move(l), 0, 0, width); }
    static Scheme occurrence_halved(LetterSet l, int width = 16) {
        return Scheme(Variant::OccurrenceHalved, std::move(l), 0, 0, width);
    }
    static Scheme count(LetterSet l, unsigned b = 2, int width = 16) { return Scheme(Variant::Count, std::move(l), b, 0, width); }
    static Scheme position(LetterSet l, unsigned p = 3, int width = 16) {
        return Scheme(Variant::Position, std::move(l), 0, p, width);
    }
    static Scheme make(Variant v, LetterSet l, unsigned b = 2, unsigned p = 3, int width = 16) {
        switch (v) {
            case Variant::Occurrence: return occurrence(std::move(l), width);
            case Variant::OccurrenceHalved: return occurrence_halved(std::move(l), width);
            case Variant::Count: return count(std::move(l), b, width);
            case Variant::Position: return position(std::move(l), p, width);
        }
        throw std::invalid_argument("unknown variant");
    }
    // Scheme::letter_capacity with 16 replaced by W.
    static std::size_t letter_capacity(Variant v, unsigned b = 2, unsigned p = 3, int width = 16) {
        const int c = fpg_letter_capacity(static_cast<int32_t>(v), width, static_cast<int32_t>(b),
                                          static_cast<int32_t>(p));
        if (c < 0) throw std::invalid_argument("invalid scheme parameters for width " + std::to_string(width));
        return static_cast<std::size_t>(c);
    }

    [[nodiscard]] Variant variant() const { return variant_; }
    [[nodiscard]] const LetterSet& letters() const { return letters_; }
    [[nodiscard]] unsigned bits_per_count() const { return b_; }
    [[nodiscard]] unsigned bits_per_position() const { return p_; }
    [[nodiscard]] int width() const { return width_; }
    [[nodiscard]] bool supports(Metric m) const { return variant_supports(variant_, m); }
    [[nodiscard]] std::size_t position_slots() const { return static_cast<std::size_t>(width_) / p_; }
    [[nodiscard]] std::size_t extra_occurrence_slots() const {
        return static_cast<std::size_t>(width_) - position_slots() * p_;
    }
    [[nodiscard]] std::size_t field_count() const {
        switch (variant_) {
            case Variant::Occurrence: return static_cast<std::size_t>(width_);
            case Variant::OccurrenceHalved: return static_cast<std::size_t>(width_) / 2;
            case Variant::Count: return static_cast<std::size_t>(width_) / b_;
            case Variant::Position: return position_slots() + extra_occurrence_slots();
        }
        return 0;
    }
    [[nodiscard]] unsigned field_width(std::size_t i) const {
        switch (variant_) {
            case Variant::Occurrence: return 1;
            case Variant::OccurrenceHalved: return 2;
            case Variant::Count: return b_;
            case Variant::Position: return i < position_slots() ? p_ : 1;
        }
        return 0;
    }
    // slot 0 owns the most significant field
    [[nodiscard]] unsigned field_shift(std::size_t i) const {
        const unsigned W = static_cast<unsigned>(width_);
        if (variant_ == Variant::Position) {
            if (i < position_slots()) return W - p_ * static_cast<unsigned>(i + 1);
            return static_cast<unsigned>(extra_occurrence_slots() - 1 - (i - position_slots()));
        }
        return W - field_width(0) * static_cast<unsigned>(i + 1);
    }

    [[nodiscard]] fpg_scheme c_struct() const {
        fpg_scheme s{};
        s.variant = static_cast<int32_t>(variant_);
        s.width = width_;
        s.bits_per_count = static_cast<int32_t>(b_);
        s.bits_per_position = static_cast<int32_t>(p_);
        s.nletters = static_cast<int32_t>(letters_.size());
        for (std::size_t i = 0; i < letters_.size() && i < 64; ++i) s.letters[i] = letters_.symbol(i);
        return s;
    }

private:
    Scheme(Variant v, LetterSet l, unsigned b, unsigned p, int width)
        : variant_(v), letters_(std::move(l)), b_(b), p_(p), width_(width) {
        if (letters_.size() > 64) throw std::invalid_argument("at most 64 letters");
        const fpg_scheme s = c_struct();
        detail::check(fpg_scheme_validate(&s));
    }
    Variant variant_;
    LetterSet letters_;
    unsigned b_, p_;
    int width_;
};

// ComparisonTables (fingerprint.hpp:171-214) generalised to W.  F_D of two
// fingerprints: the popcount of their xor for occurrence / halved, the number
// of fields with a non-zero xor for count / position (a +-1 counter step can
// flip every bit of its field, so a field counts once).  At W = 16 the
// reference's 2^16-entry tables are built; at W = 32 / 64 the same values
// come from per-field masks (a table would not fit).
class ComparisonTables {
public:
    explicit ComparisonTables(const Scheme& scheme) : width_(scheme.width()) {
        for (unsigned d = 0; d < ceil_half_.size(); ++d) ceil_half_[d] = static_cast<std::uint8_t>((d + 1) / 2);
        const Variant v = scheme.variant();
        fields_ = v == Variant::Count || v == Variant::Position;
        if (fields_)
            for (std::size_t i = 0; i < scheme.field_count(); ++i) {
                const unsigned w = scheme.field_width(i);
                masks_.push_back((w >= 64 ? ~0ull : ((1ull << w) - 1)) << scheme.field_shift(i));
            }
        if (width_ == 16) {
            popcount_.resize(1u << 16);
            for (std::uint32_t x = 0; x < popcount_.size(); ++x)
                popcount_[x] = static_cast<std::uint8_t>(std::popcount(x));
            if (fields_) {
                groups_.resize(1u << 16);
                for (std::uint32_t x = 0; x < groups_.size(); ++x) groups_[x] = static_cast<std::uint8_t>(fold(x));
            }
        }
    }

    [[nodiscard]] int width() const { return width_; }
    [[nodiscard]] int popcount16(std::uint16_t x) const {
        return popcount_.empty() ? std::popcount(x) : popcount_[x];
    }
    [[nodiscard]] int ceil_half(int d) const { return ceil_half_[static_cast<std::size_t>(d)]; }
    /// Mismatching-field count for an xor value (count / position schemes).
    [[nodiscard]] int group_mismatch(std::uint64_t x) const {
        return groups_.empty() ? fold(x) : groups_[static_cast<std::uint16_t>(x)];
    }
    [[nodiscard]] bool has_group_table() const { return fields_; }
    /// Fingerprint distance of the scheme these tables were built for.
    [[nodiscard]] int distance(Fingerprint a, Fingerprint b) const {
        const std::uint64_t x = a.bits ^ b.bits;
        if (fields_) return group_mismatch(x);
        return width_ == 16 ? popcount_[static_cast<std::uint16_t>(x)] : std::popcount(x);
    }

private:
    [[nodiscard]] int fold(std::uint64_t x) const {
        int m = 0;
        for (const std::uint64_t mask : masks_) m += (x & mask) != 0;
        return m;
    }
    int width_;
    bool fields_ = false;
    std::vector<std::uint64_t> masks_;
    std::vector<std::uint8_t> popcount_, groups_;
    std::array<std::uint8_t, 65> ceil_half_{};
};

/// Fingerprint distance F_D (fingerprint.hpp:287-291).
inline int fingerprint_distance(Fingerprint f1, Fingerprint f2, const Scheme&, const ComparisonTables& tables) {
    return tables.distance(f1, f2);
}

/// Lower bound on the true number of errors: ceil(F_D / 2) (fingerprint.hpp:293-296).
inline int lower_bound_errors(int fd, const ComparisonTables& tables) { return tables.ceil_half(fd); }

/// True when the fingerprints alone prove the distance exceeds k (fingerprint.hpp:298-301).
inline bool can_reject(Fingerprint f1, Fingerprint f2, int k, const Scheme& scheme, const ComparisonTables& tables) {
    return lower_bound_errors(fingerprint_distance(f1, f2, scheme, tables), tables) > k;
}

inline SymbolFrequencyTable compute_frequencies_gpu(std::string_view text, int device) {
    SymbolFrequencyTable t;
    std::uint64_t counts[256] = {0};
    detail::check(fpg_byte_histogram(reinterpret_cast<const std::uint8_t*>(text.data()), text.size(), device, counts));
    for (int c = 0; c < 256; ++c) t.counts[static_cast<std::size_t>(c)] = counts[c];
    t.total = text.size();
    return t;
}

// build() for a batch of strings, on `device` (K1).
inline std::vector<Fingerprint> build_many(const std::vector<std::string>& words, const Scheme& scheme,
                                           int device = 0) {
    std::vector<std::uint64_t> offs(words.size() + 1, 0);
    std::string blob;
    for (std::size_t i = 0; i < words.size(); ++i) {
        blob += words[i];
        offs[i + 1] = blob.size();
    }
    std::vector<std::uint64_t> out(words.size());
    const fpg_scheme s = scheme.c_struct();
    detail::check(fpg_build_fingerprints(reinterpret_cast<const std::uint8_t*>(blob.data()), offs.data(),
                                         words.size(), &s, device, out.data()));
    std::vector<Fingerprint> r(words.size());
    for (std::size_t i = 0; i < words.size(); ++i) r[i].bits = out[i];
    return r;
}

inline Fingerprint build(std::string_view s, const Scheme& scheme, int device = 0) {
    return build_many({std::string(s)}, scheme, device)[0];
}

// Slot-0 field leftmost; fields space-separated except for occurrence.
inline std::string render(Fingerprint f, const Scheme& scheme) {
    std::string out;
    for (std::size_t i = 0; i < scheme.field_count(); ++i) {
        if (i != 0 && scheme.variant() != Variant::Occurrence) out.push_back(' ');
        const unsigned w = scheme.field_width(i), sh = scheme.field_shift(i);
        for (unsigned b = 0; b < w; ++b) out.push_back(((f.bits >> (sh + w - 1 - b)) & 1u) ? '1' : '0');
    }
    return out;
}

}  // namespace fingerprints
