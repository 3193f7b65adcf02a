// gpu_letters.hpp -- alphabet model of the B200 build (host only).
//
// Mirrors the reference's letter_model.hpp interface (SymbolFrequencyTable
// :15-31, compute_frequencies :33-45, LetterStrategy :47, LetterSet :60-87,
// select_letters :94-134) so reference callers compile unchanged.  Letter
// selection is host bookkeeping done once per dictionary; nothing here is on
// the per-pair path.
#pragma once

#include <algorithm>
#include <array>
#include <cstddef>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <string_view>
#include <vector>

namespace fingerprints {

struct SymbolFrequencyTable {
    std::array<std::uint64_t, 256> counts{};
    std::uint64_t total = 0;

    void add(std::string_view text) {
        for (unsigned char c : text) counts[c] += 1;
        total += text.size();
    }
    [[nodiscard]] std::size_t alphabet_size() const {
        return static_cast<std::size_t>(std::count_if(counts.begin(), counts.end(),
                                                      [](std::uint64_t v) { return v != 0; }));
    }
};

inline SymbolFrequencyTable compute_frequencies(std::string_view text) {
    SymbolFrequencyTable t;
    t.add(text);
    return t;
}

inline SymbolFrequencyTable compute_frequencies(const std::vector<std::string>& words) {
    SymbolFrequencyTable t;
    for (const std::string& w : words) t.add(w);
    return t;
}

// compute_frequencies of a large blob on the GPU (libfpg.so).
inline SymbolFrequencyTable compute_frequencies_gpu(std::string_view text, int device = 0);

enum class LetterStrategy { Common, Mixed, Rare };

inline std::string_view to_string(LetterStrategy s) {
    return s == LetterStrategy::Common ? "common" : s == LetterStrategy::Mixed ? "mixed" : "rare";
}

// Ordered symbol subset; slot(c) = position of byte c, or -1.
class LetterSet {
public:
    LetterSet() { slots_.fill(-1); }
    explicit LetterSet(std::string_view symbols) : symbols_(symbols) {
        slots_.fill(-1);
        for (std::size_t i = 0; i < symbols_.size(); ++i) {
            auto& s = slots_[static_cast<unsigned char>(symbols_[i])];
            if (s >= 0) throw std::invalid_argument("LetterSet: duplicate symbol in letter set");
            s = static_cast<std::int16_t>(i);
        }
    }
    [[nodiscard]] std::size_t size() const { return symbols_.size(); }
    [[nodiscard]] unsigned char symbol(std::size_t slot) const {
        return static_cast<unsigned char>(symbols_[slot]);
    }
    [[nodiscard]] int slot_of(unsigned char c) const { return slots_[c]; }
    [[nodiscard]] bool contains(unsigned char c) const { return slots_[c] >= 0; }
    [[nodiscard]] const std::string& symbols() const { return symbols_; }

private:
    std::string symbols_;
    std::array<std::int16_t, 256> slots_{};
};

// Symbols ranked by (count, byte) ascending; common = highest, rare = lowest,
// mixed = ceil(n/2) common + floor(n/2) rare.
inline LetterSet select_letters(const SymbolFrequencyTable& freq, std::size_t count, LetterStrategy strategy) {
    std::vector<unsigned char> order;
    for (int c = 0; c < 256; ++c)
        if (freq.counts[static_cast<std::size_t>(c)]) order.push_back(static_cast<unsigned char>(c));
    std::stable_sort(order.begin(), order.end(), [&](unsigned char a, unsigned char b) {
        return freq.counts[a] < freq.counts[b];
    });
    if (order.size() < count)
        throw std::invalid_argument("select_letters: collection has " + std::to_string(order.size()) +
                                    " distinct symbols, need " + std::to_string(count));
    std::string out;
    const std::size_t top = strategy == LetterStrategy::Common ? count
                          : strategy == LetterStrategy::Rare   ? 0
                                                               : (count + 1) / 2;
    for (std::size_t i = 0; i < top; ++i) out.push_back(static_cast<char>(order[order.size() - 1 - i]));
    for (std::size_t i = 0; i < count - top; ++i) out.push_back(static_cast<char>(order[i]));
    return LetterSet(out);
}

inline std::string_view english_default_letters() { return "etaoinshrdlcumwfgypbvkjxqz"; }

}  // namespace fingerprints
