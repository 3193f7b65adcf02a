// fpg_kernels.cuh -- sm_100a kernels of the fingerprint-filtered k<=1 scan.
//
//   K1 k_build      one thread per string: fingerprint (reference build(),
//                   fingerprint.hpp:216-284, generalised to W bits) + copy of
//                   the bytes into the length-bucketed, 16-byte-stride layout.
//   K2 k_scan       query x word tiles of one (query length, word length)
//                   bucket pair: XOR + POPC fingerprint test
//                   (dictionary.hpp:102-106; ComparisonTables::distance
//                   fingerprint.hpp:171-214) for every pair, survivors
//                   compacted per warp with __ballot_sync into shared memory
//                   and verified there at k<=1 (edit_distance.hpp:18-64),
//                   matches appended with warp-aggregated atomics.
//   K4 k_offsets / k_low_ids   CSR of the radix-sorted (query, word) keys.
#pragma once

#include <cstdint>

namespace fpg {

constexpr int kMaxLen = 4096;

// Symbol -> slot table and scheme constants.  Passed by value as a kernel
// parameter, i.e. it lives in the constant bank; K1 copies the table into
// shared memory because lanes index it with divergent bytes.
struct SchemeParams {
    int8_t slot[256];
    int32_t variant, width, b, p, nletters, slots, extra;
    int32_t onehot;        // count, W=16, b=2: K2 compares a 32-bit one-hot form
    uint64_t mask_fold;    // bit at the LSB of every multi-bit field (count / position)
    uint64_t mask_single;  // 1-bit fields of the position layout (extra letters)
    uint64_t full;         // W low bits set
};

// One (query range) x (word range) block of work; both ranges lie in one
// length bucket of their collection, so the pair's length relation (equal,
// word longer by one, word shorter by one, or incompatible) is tile-uniform.
struct Tile {
    uint32_t q_begin, q_count;   // sorted positions in the query collection
    uint32_t w_begin, w_count;   // sorted positions in the dictionary
    uint64_t q_bytes, w_bytes;   // byte offset of q_begin / w_begin in the padded blobs
    uint16_t q_len, w_len, q_stride, w_stride;
    uint32_t count_only, pad;    // count_only: survivors counted, never verified
};

struct ScanParams {
    const uint64_t* q_fp;       // query comparison words (fingerprint or its one-hot form), sorted order
    const uint8_t* q_bytes;     // padded query bytes
    const uint32_t* q_ids;      // sorted position -> input query index
    const uint64_t* w_fp;
    const uint8_t* w_bytes;
    const uint32_t* w_ids;      // sorted position -> input word index (shard-local)
    uint64_t id_base;           // added to word ids
    uint32_t* q_survivors;      // per input query: pairs passing the fingerprint test
    unsigned long long* out;    // (query << 32 | word) match keys
    unsigned long long* out_count;
    unsigned long long* survivors_total;
    uint64_t out_cap;
    uint64_t mask_fold, mask_single;
    int32_t thr;                // reject iff F_D > thr (= 2k), thr huge when !use_filter
    int32_t k;
    int32_t fold;               // field width for the generic fold (kGeneric only)
    const uint32_t* q_sig;      // occurrence signatures (verifier pre-check)
    const uint32_t* w_sig;
};

__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31; }

// ---------------------------------------------------------------- K1 build
template <int VARIANT>
__device__ __forceinline__ uint64_t build_fp(const uint8_t* s, int n, const int8_t* slot,
                                             const SchemeParams& P) {
    const int W = P.width;
    uint64_t bits = 0;
    if (VARIANT == 0) {                                  // build_occurrence :216-224
        for (int i = 0; i < n; ++i) {
            int q = slot[s[i]];
            if (q >= 0) bits |= 1ull << (W - 1 - q);
        }
    } else if (VARIANT == 1) {                           // build_occurrence_halved :226-238
        const int half = n >> 1;
        for (int i = 0; i < n; ++i) {
            int q = slot[s[i]];
            if (q >= 0) bits |= 1ull << (i < half ? W - 1 - 2 * q : W - 2 - 2 * q);
        }
    } else if (VARIANT == 2) {                           // build_count :240-254
        const int b = P.b;
        const uint64_t sat = (1ull << b) - 1;
        for (int i = 0; i < n; ++i) {
            int q = slot[s[i]];
            if (q < 0) continue;
            const int shift = W - b * (q + 1);
            if (((bits >> shift) & sat) != sat) bits += 1ull << shift;
        }
    } else {                                             // build_position :256-274 (one pass)
        const int p = P.p;
        const uint64_t absent = (1ull << p) - 1;
        uint64_t seen = 0;                               // letters already placed (<= 64)
        for (int q = 0; q < P.slots; ++q) bits |= absent << (W - p * (q + 1));
        for (int i = 0; i < n; ++i) {
            int q = slot[s[i]];
            if (q < 0 || ((seen >> q) & 1)) continue;
            seen |= 1ull << q;
            if (q < P.slots) {
                const int shift = W - p * (q + 1);
                if ((uint64_t)i < absent) bits = (bits & ~(absent << shift)) | ((uint64_t)i << shift);
            } else {
                bits |= 1ull << (P.extra - 1 - (q - P.slots));
            }
        }
    }
    return bits;
}

// Comparison form of a count-16 (b=2) fingerprint: field i (value v in 0..3)
// becomes bit 4i+v of a 32-bit word, so popc(a ^ b) = 2 * (number of
// differing fields) = 2 * F_D (ComparisonTables group count,
// fingerprint.hpp:180-192) with one XOR + one POPC and no fold.
__device__ __forceinline__ uint64_t onehot_count16(uint64_t fp) {
    uint32_t r = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) r |= 1u << (4 * i + (int)((fp >> (14 - 2 * i)) & 3u));
    return r;
}

// Occurrence signature of a string: bit (c & 31) for every byte c.  One edit
// changes at most two of its bits, so popc(sig_a ^ sig_b) > 2 proves
// distance > 1 (hence > k for k <= 1) for Hamming and Levenshtein alike (the occurrence bound of
// fingerprint.hpp:216-224 over a 32-letter hashed alphabet).  K2's verifier
// uses it as an exact pre-check before comparing bytes.
__device__ __forceinline__ uint32_t occurrence_sig(const uint8_t* s, int n) {
    uint32_t g = 0;
    for (int i = 0; i < n; ++i) g |= 1u << (s[i] & 31);
    return g;
}

// Inputs: raw blob + offsets, `order` = sorted position -> input index (stable
// sort by length), per-length bucket tables.  Outputs per sorted position:
// fingerprint, input id, and the bytes at the bucket's fixed stride (zero
// padded to the stride).
template <int VARIANT>
__global__ void __launch_bounds__(256) k_build(const uint8_t* __restrict__ blob,
                                               const uint64_t* __restrict__ offsets,
                                               const uint32_t* __restrict__ order, uint64_t n,
                                               const uint32_t* __restrict__ bucket_start,
                                               const uint64_t* __restrict__ bucket_bytes,
                                               const __grid_constant__ SchemeParams P,
                                               uint64_t* __restrict__ fp_out,
                                               uint64_t* __restrict__ cmp_out,
                                               uint32_t* __restrict__ sig_out,
                                               uint32_t* __restrict__ id_out,
                                               uint8_t* __restrict__ bytes_out) {
    __shared__ int8_t s_slot[256];
    s_slot[threadIdx.x] = P.slot[threadIdx.x];           // blockDim == 256
    __syncthreads();
    const uint64_t pos = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (pos >= n) return;
    const uint32_t id = order ? order[pos] : (uint32_t)pos;
    const uint64_t beg = offsets[id];
    const int len = (int)(offsets[id + 1] - beg);
    const uint8_t* s = blob + beg;
    const uint64_t fp = build_fp<VARIANT>(s, len, s_slot, P);
    fp_out[pos] = fp;
    if (cmp_out) cmp_out[pos] = P.onehot ? onehot_count16(fp) : fp;
    if (sig_out) sig_out[pos] = occurrence_sig(s, len);
    if (id_out) id_out[pos] = id;
    if (bytes_out) {
        const int stride = len <= 16 ? 16 : (len + 15) & ~15;
        uint8_t* dst = bytes_out + bucket_bytes[len] + (uint64_t)(pos - bucket_start[len]) * stride;
        // dst is 16-byte aligned: assemble 16-byte chunks in registers.
        for (int c = 0; c < stride; c += 16) {
            uint32_t w[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                uint32_t v = 0;
#pragma unroll
                for (int t = 0; t < 4; ++t) {
                    const int i = c + 4 * j + t;
                    if (i < len) v |= (uint32_t)s[i] << (8 * t);
                }
                w[j] = v;
            }
            *reinterpret_cast<uint4*>(dst + c) = make_uint4(w[0], w[1], w[2], w[3]);
        }
    }
}

__global__ void k_lengths(const uint64_t* __restrict__ offsets, uint64_t n,
                          uint16_t* __restrict__ len_out, uint32_t* __restrict__ idx_out,
                          uint32_t* __restrict__ hist, uint32_t* __restrict__ too_long) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    uint64_t len = offsets[i + 1] - offsets[i];
    if (len > (uint64_t)kMaxLen) {
        atomicAdd(too_long, 1u);
        len = kMaxLen;
    }
    len_out[i] = (uint16_t)len;
    idx_out[i] = (uint32_t)i;
    atomicAdd(&hist[len], 1u);
}

__global__ void k_scatter_prints(const uint64_t* __restrict__ fp, const uint32_t* __restrict__ ids,
                                 uint64_t n, uint64_t* __restrict__ out) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[ids[i]] = fp[i];
}

// ---------------------------------------------------------------- K4 CSR
// offsets[q] = lower_bound(keys, q << 32) for q in [0, nq]; keys sorted.
__global__ void k_offsets(const unsigned long long* __restrict__ keys, uint64_t total, uint64_t nq,
                          uint64_t* __restrict__ offsets) {
    const uint64_t q = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (q > nq) return;
    const unsigned long long key = (unsigned long long)q << 32;
    uint64_t lo = 0, hi = total;
    while (lo < hi) {
        const uint64_t mid = (lo + hi) >> 1;
        if (keys[mid] < key) lo = mid + 1;
        else hi = mid;
    }
    offsets[q] = lo;
}

__global__ void k_low_ids(const unsigned long long* __restrict__ keys, uint64_t total,
                          uint32_t* __restrict__ ids) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < total) ids[i] = (uint32_t)keys[i];
}

}  // namespace fpg

#include "fpg_scan.cuh"
