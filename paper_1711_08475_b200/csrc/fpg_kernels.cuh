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
    const uint64_t* q_fp;       // query fingerprints, sorted order
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
    fp_out[pos] = build_fp<VARIANT>(s, len, s_slot, P);
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

// ---------------------------------------------------------------- K2 scan

// F_D of the scheme (ComparisonTables::distance, fingerprint.hpp:205-207):
// popcount for occurrence / halved, number of non-zero fields otherwise.
template <int VARIANT, int W>
__device__ __forceinline__ int fp_distance(uint64_t x, uint64_t mask_fold, uint64_t mask_single,
                                           int fold) {
    if (W <= 32) {
        const uint32_t y = (uint32_t)x;
        if (VARIANT <= 1) return __popc(y);
        uint32_t f = y;
        if (VARIANT == 2) {
#pragma unroll 4
            for (int j = 1; j < fold; ++j) f |= y >> j;
            return __popc(f & (uint32_t)mask_fold);
        }
#pragma unroll 4
        for (int j = 1; j < fold; ++j) f |= y >> j;
        return __popc((f & (uint32_t)mask_fold) | (y & (uint32_t)mask_single));
    } else {
        if (VARIANT <= 1) return __popcll(x);
        uint64_t f = x;
#pragma unroll 4
        for (int j = 1; j < fold; ++j) f |= x >> j;
        if (VARIANT == 2) return __popcll(f & mask_fold);
        return __popcll((f & mask_fold) | (x & mask_single));
    }
}

__device__ __forceinline__ uint32_t ld32(const uint8_t* base, int chunk, int stride) {
    return (4 * chunk < stride) ? __ldg(reinterpret_cast<const uint32_t*>(base) + chunk) : 0u;
}

// k<=1 verifier for one (query, word) pair whose byte strings are zero-padded
// to their strides.  Semantics of hamming_bounded / levenshtein_bounded
// (edit_distance.hpp:18-64) at k in {0,1}:
//   equal lengths: distance <= 1  <=>  first mismatching byte == last one;
//   lengths differ by one (long s, short t): t is s with one byte deleted  <=>
//   (last mismatch of t vs s shifted by one) < (first mismatch of t vs s).
__device__ __forceinline__ bool verify_pair(const uint8_t* q, int m, int qs, const uint8_t* w,
                                            int n, int ws, int k) {
    const int d = n - m;
    if (d == 0) {
        const int nc = (m + 3) >> 2;
        int first = 1 << 30, last = -1;
        for (int c = 0; c < nc; ++c) {
            const uint32_t x = ld32(q, c, qs) ^ ld32(w, c, ws);
            if (x) {
                if (first == (1 << 30)) first = 4 * c + ((__ffs(x) - 1) >> 3);
                last = 4 * c + ((31 - __clz(x)) >> 3);
                if (k == 0 || last != first) return false;
            }
        }
        return true;
    }
    if (k == 0) return false;
    // s = longer string, t = shorter string
    const uint8_t* s = d > 0 ? w : q;
    const uint8_t* t = d > 0 ? q : w;
    const int ss = d > 0 ? ws : qs, ts = d > 0 ? qs : ws;
    const int nc = ((d > 0 ? n : m) + 3) >> 2;
    int firstA = 1 << 30, lastB = -1;
    uint32_t s0 = ld32(s, 0, ss);
    for (int c = 0; c < nc; ++c) {
        const uint32_t s1 = ld32(s, c + 1, ss);
        const uint32_t tc = ld32(t, c, ts);
        const uint32_t xa = tc ^ s0;
        const uint32_t xb = tc ^ __funnelshift_r(s0, s1, 8);
        if (xa && firstA == (1 << 30)) firstA = 4 * c + ((__ffs(xa) - 1) >> 3);
        if (xb) lastB = 4 * c + ((31 - __clz(xb)) >> 3);
        s0 = s1;
    }
    return lastB < firstA;
}

constexpr int kScanThreads = 256;
constexpr int kWordsPerThread = 4;                       // R
constexpr int kTileWords = kScanThreads * kWordsPerThread;
constexpr int kTileQueries = 256;
constexpr int kQueueCap = 512;                           // candidates per warp

template <int VARIANT, int W>
__global__ void __launch_bounds__(kScanThreads) k_scan(const Tile* __restrict__ tiles,
                                                       uint32_t ntiles,
                                                       const __grid_constant__ ScanParams P,
                                                       int fold) {
    using FP = typename std::conditional<(W <= 32), uint32_t, uint64_t>::type;
    __shared__ FP s_qfp[kTileQueries];
    __shared__ uint32_t s_qsurv[kTileQueries];
    __shared__ uint32_t s_queue[kScanThreads / 32][kQueueCap];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t lt_mask = (1u << lane) - 1u;
    uint32_t* queue = s_queue[warp];

    for (uint32_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const Tile T = tiles[t];
        __syncthreads();  // previous tile's shared state fully consumed
        for (uint32_t i = tid; i < T.q_count; i += kScanThreads) {
            s_qfp[i] = (FP)P.q_fp[T.q_begin + i];
            s_qsurv[i] = 0;
        }
        FP wf[kWordsPerThread];
        bool wv[kWordsPerThread];
#pragma unroll
        for (int r = 0; r < kWordsPerThread; ++r) {
            const uint32_t widx = r * kScanThreads + tid;
            wv[r] = widx < T.w_count;
            wf[r] = wv[r] ? (FP)P.w_fp[T.w_begin + widx] : (FP)0;
        }
        __syncthreads();

        const uint8_t* qbase = P.q_bytes + T.q_bytes;
        const uint8_t* wbase = P.w_bytes + T.w_bytes;
        int qn = 0;  // warp-uniform queue fill

        auto flush = [&]() {
            __syncwarp();
            for (int base = 0; base < qn; base += 32) {
                const int c = base + lane;
                bool hit = false;
                uint32_t e = 0;
                if (c < qn) {
                    e = queue[c];
                    const uint32_t j = e >> 16, widx = e & 0xffffu;
                    hit = verify_pair(qbase + (uint64_t)j * T.q_stride, T.q_len, T.q_stride,
                                      wbase + (uint64_t)widx * T.w_stride, T.w_len, T.w_stride, P.k);
                }
                const uint32_t hb = __ballot_sync(0xffffffffu, hit);
                if (hb) {
                    unsigned long long slot = 0;
                    if (lane == 0) slot = atomicAdd(P.out_count, (unsigned long long)__popc(hb));
                    slot = __shfl_sync(0xffffffffu, slot, 0);
                    if (hit) {
                        const uint64_t o = slot + __popc(hb & lt_mask);
                        if (o < P.out_cap) {
                            const uint32_t j = e >> 16, widx = e & 0xffffu;
                            const uint64_t qid = P.q_ids[T.q_begin + j];
                            const uint64_t wid = P.id_base + P.w_ids[T.w_begin + widx];
                            P.out[o] = (qid << 32) | wid;
                        }
                    }
                }
            }
            __syncwarp();
            qn = 0;
        };

        for (uint32_t j = 0; j < T.q_count; ++j) {
            const FP qf = s_qfp[j];
            bool pass[kWordsPerThread];
            bool any = false;
#pragma unroll
            for (int r = 0; r < kWordsPerThread; ++r) {
                pass[r] = wv[r] &&
                          fp_distance<VARIANT, W>((uint64_t)(qf ^ wf[r]), P.mask_fold, P.mask_single,
                                                  fold) <= P.thr;
                any |= pass[r];
            }
            if (!__any_sync(0xffffffffu, any)) continue;
            uint32_t tot = 0;
#pragma unroll
            for (int r = 0; r < kWordsPerThread; ++r) {
                const uint32_t b = __ballot_sync(0xffffffffu, pass[r]);
                if (!T.count_only && pass[r])
                    queue[qn + __popc(b & lt_mask)] = (j << 16) | (uint32_t)(r * kScanThreads + tid);
                qn += __popc(b);
                tot += __popc(b);
            }
            if (lane == 0) atomicAdd(&s_qsurv[j], tot);
            if (T.count_only) qn = 0;
            else if (qn > kQueueCap - 32 * kWordsPerThread) flush();
        }
        if (!T.count_only) flush();
        __syncthreads();
        unsigned long long local = 0;
        for (uint32_t i = tid; i < T.q_count; i += kScanThreads) {
            const uint32_t v = s_qsurv[i];
            if (v) {
                atomicAdd(&P.q_survivors[P.q_ids[T.q_begin + i]], v);
                local += v;
            }
        }
        // one atomic per warp for the run total
        for (int o = 16; o; o >>= 1) local += __shfl_xor_sync(0xffffffffu, local, o);
        if (lane == 0 && local) atomicAdd(P.survivors_total, local);
    }
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
