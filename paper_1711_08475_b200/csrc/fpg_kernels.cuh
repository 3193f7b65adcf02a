// fpg_kernels.cuh -- sm_100a kernels of the fingerprint-filtered k-approximate scan.
//
//   K0 k_hist256    byte histogram (sig' ranking, letter selection)
//   K1 k_build      one thread per string: fingerprint (reference build(),
//                   fingerprint.hpp:216-284, generalised to W bits), sig'
//                   code, group weights, and the bytes copied into the
//                   length-bucketed 16-byte-stride layout.  k_weight_keys /
//                   k_lengths feed the (length, group weights) sort of the
//                   dictionary.
//   K1b k_planes    bit-sliced planes and group-weight box per 32-word slab
//                   (fpg_slice.cuh)
//   K2 k_slice      the bit-sliced filter + k <= 1 verifier (fpg_slice.cuh);
//      k_scan       the generic per-pair XOR + POPC filter (fpg_scan.cuh):
//                   fields wider than 4 bits, k >= 2 (banded verifier)
//   K4 k_seg_scatter / k_seg_sort   CSR: keys scattered into per-query
//                   segments (sorted word positions mapped to input-order
//                   ids), segments of <= 32 warp-sorted (larger ones: CUB
//                   segmented sort, launched by the host)
#pragma once

#include <cstdint>

namespace fpg {

constexpr int kMaxLen = 4096;
// Words of at most kXLen bytes get exact position-code planes (K2's exact
// Hamming path, fpg_slice.cuh): 5 bits per position.
constexpr int kXLen = 6;
constexpr int kXBits = 5;

// Symbol -> slot table and scheme constants.  Passed by value as a kernel
// parameter, i.e. it lives in the constant bank; K1 copies the table into
// shared memory because lanes index it with divergent bytes.
struct SchemeParams {
    int8_t slot[256];
    int8_t sigbit[256];    // sig' field of a non-letter byte (fpg_slice.cuh), or -1
    uint8_t xcode[256];    // exact path: dense code of a dictionary byte (< 31); 31 for bytes the dictionary lacks
    int32_t xlen;          // exact path on (kXLen) or off (0)
    int32_t nsig;          // sig' fields S
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
    unsigned long long* out_count;  // key slots reserved (OutChunk)
    unsigned long long* match_total;
    unsigned long long* survivors_total;
    uint64_t out_cap;
    uint64_t mask_fold, mask_single;
    int32_t thr;                // reject iff F_D > thr (= 2k), thr huge when !use_filter
    int32_t k;
    int32_t fold;               // field width for the generic fold (kGeneric only)
    const uint32_t* q_sig;      // occurrence signatures (verifier pre-check)
    const uint32_t* w_sig;
    int32_t sig_on;             // signature pre-check (exact for k <= 1 only)
    int32_t lev;                // metric is Levenshtein (k >= 2 verifier)
    uint32_t* q_matches;        // per input query: matches (K4 segment sizes)
};

__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31; }

// ---------------------------------------------------------------- K1 build
// Incremental fingerprint builder: one call per letter occurrence (slot q of
// byte i of an n-byte string), the reference builders generalised to W bits.
template <int VARIANT>
struct FpBuilder {
    uint64_t bits = 0;
    uint64_t seen = 0;  // position: letters already placed (<= 64 letters)

    __device__ __forceinline__ void init(const SchemeParams& P) {
        if (VARIANT == 3) {                              // build_position :258: every field starts absent
            const uint64_t absent = (1ull << P.p) - 1;
            for (int q = 0; q < P.slots; ++q) bits |= absent << (P.width - P.p * (q + 1));
        }
    }
    __device__ __forceinline__ void add(int q, int i, int n, const SchemeParams& P) {
        const int W = P.width;
        if (VARIANT == 0) {                              // build_occurrence :216-224
            bits |= 1ull << (W - 1 - q);
        } else if (VARIANT == 1) {                       // build_occurrence_halved :226-238 (half = n / 2)
            bits |= 1ull << (i < (n >> 1) ? W - 1 - 2 * q : W - 2 - 2 * q);
        } else if (VARIANT == 2) {                       // build_count :240-254 (saturating b-bit counter)
            const uint64_t sat = (1ull << P.b) - 1;
            const int shift = W - P.b * (q + 1);
            if (((bits >> shift) & sat) != sat) bits += 1ull << shift;
        } else {                                         // build_position :256-274, one pass
            if ((seen >> q) & 1) return;                 // first occurrence only
            seen |= 1ull << q;
            if (q < P.slots) {
                const uint64_t absent = (1ull << P.p) - 1;
                const int shift = W - P.p * (q + 1);
                if ((uint64_t)i < absent) bits = (bits & ~(absent << shift)) | ((uint64_t)i << shift);
            } else {
                bits |= 1ull << (P.extra - 1 - (q - P.slots));
            }
        }
    }
};

// Bytes [at, at + rem) of `blob` (rem <= 16, zero beyond) as four little-endian
// words: five independent aligned 4-byte loads and funnel shifts, so a string
// costs one memory latency per 16 bytes.  Blobs carry >= 16 bytes of tail padding.
__device__ __forceinline__ void load_chunk(const uint8_t* blob, uint64_t at, int rem, uint32_t (&w)[4]) {
    const uint64_t base = at & ~3ull;
    const uint32_t sh = (uint32_t)(at & 3) * 8;
    const int need = (int)((at & 3) + rem + 3) >> 2;     // words overlapping the range
    const uint32_t* p = reinterpret_cast<const uint32_t*>(blob + base);
    uint32_t v[5];
#pragma unroll
    for (int j = 0; j < 5; ++j) v[j] = j < need ? __ldg(p + j) : 0u;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const uint32_t x = __funnelshift_r(v[j], v[j + 1], sh);
        const int keep = rem - 4 * j;                    // bytes of this word inside the string
        w[j] = keep >= 4 ? x : keep <= 0 ? 0u : (x & ((1u << (8 * keep)) - 1u));
    }
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

// Group weights: the fields are dealt round robin into kGroups = 8 groups
// (field i -> group i & 7; occurrence / halved: bit i, count / position: the
// extra one-bit fields, then the multi-bit fields), and nibble g of the
// result is the number of "present" fields of group g (occurrence / halved:
// set bits; count: non-zero counters; position: letters whose first position
// is recorded, plus the extra occurrence bits; at most 8 per group for
// W <= 64).  One differing field changes one group's weight by at most one, so
//   sum_g |gw_g(a) - gw_g(b)| <= F_D          (fingerprint.hpp:171-214)
// and K2 skips query / word groups whose group-weight boxes are more than 2k
// apart (L1 distance).
constexpr int kGroups = 8;
__device__ __forceinline__ uint32_t fp_gweight(uint64_t fp, const SchemeParams& P) {
    if (P.variant == 0 || P.variant == 1) {
        uint32_t w = 0;
#pragma unroll
        for (int g = 0; g < kGroups; ++g) w |= (uint32_t)__popcll(fp & (0x0101010101010101ull << g)) << (4 * g);
        return w;
    }
    const int fw = P.variant == 2 ? P.b : P.p;
    const int nf = P.variant == 2 ? P.width / P.b : P.slots;
    const int extra = P.variant == 2 ? 0 : P.extra;
    const uint64_t fmask = fw >= 64 ? ~0ull : ((1ull << fw) - 1);
    uint32_t w = 0;
    for (int e = 0; e < extra; ++e) w += (uint32_t)((fp >> e) & 1u) << (4 * (e & 7));
    for (int f = 0; f < nf; ++f) {
        const uint64_t v = (fp >> (P.width - fw * (f + 1))) & fmask;
        const bool present = P.variant == 2 ? (v != 0) : (v != fmask);  // position: all-ones = absent
        w += (uint32_t)present << (4 * ((extra + f) & 7));
    }
    return w;
}

// Sort keys of the dictionary's K2 layout: length << 32 | the group weights
// with group 0 in the most significant nibble, per word in input order (the
// fingerprint is computed here and again by k_build).
template <int VARIANT>
__global__ void __launch_bounds__(256) k_weight_keys(const uint8_t* __restrict__ blob,
                                                     const uint64_t* __restrict__ offsets, uint64_t n,
                                                     const __grid_constant__ SchemeParams P,
                                                     uint64_t* __restrict__ keys) {
    __shared__ int8_t s_slot[256];
    s_slot[threadIdx.x] = P.slot[threadIdx.x];
    __syncthreads();
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint64_t beg = offsets[i];
    const uint64_t len64 = offsets[i + 1] - beg;
    const int len = len64 > (uint64_t)kMaxLen ? kMaxLen : (int)len64;
    FpBuilder<VARIANT> fb;
    fb.init(P);
    for (int c = 0; c < len; c += 16) {
        uint32_t w[4];
        const int rem = min(16, len - c);
        load_chunk(blob, beg + c, rem, w);
#pragma unroll
        for (int t = 0; t < 16; ++t)
            if (t < rem) {
                const int q = s_slot[(w[t >> 2] >> (8 * (t & 3))) & 0xffu];
                if (q >= 0) fb.add(q, c + t, len, P);
            }
    }
    const uint32_t gw = fp_gweight(fb.bits, P);
    uint32_t key = 0;
#pragma unroll
    for (int g = 0; g < kGroups; ++g) key |= ((gw >> (4 * g)) & 0xfu) << (28 - 4 * g);
    keys[i] = ((uint64_t)len << 32) | key;
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
                                               uint32_t* __restrict__ sigp_out,
                                               uint32_t* __restrict__ id_out,
                                               uint8_t* __restrict__ bytes_out,
                                               uint16_t* __restrict__ len_out = nullptr,
                                               uint32_t* __restrict__ zero_by_id = nullptr,
                                               unsigned long long* __restrict__ zero64 = nullptr,
                                               int nzero64 = 0, uint32_t* __restrict__ weight_out = nullptr,
                                               uint32_t* __restrict__ xc_out = nullptr) {
    __shared__ int8_t s_slot[256];
    __shared__ int8_t s_sigbit[256];
    __shared__ uint8_t s_xcode[256];
    s_slot[threadIdx.x] = P.slot[threadIdx.x];           // blockDim == 256
    s_sigbit[threadIdx.x] = P.sigbit[threadIdx.x];
    s_xcode[threadIdx.x] = P.xcode[threadIdx.x];
    __syncthreads();
    if (zero64 && blockIdx.x == 0 && (int)threadIdx.x < nzero64) zero64[threadIdx.x] = 0ull;
    const uint64_t pos = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (pos >= n) return;
    const uint32_t id = order ? order[pos] : (uint32_t)pos;
    const uint64_t beg = offsets[id];
    const int len = (int)(offsets[id + 1] - beg);
    if (len_out) len_out[pos] = (uint16_t)len;
    if (zero_by_id) zero_by_id[id] = zero_by_id[id + n] = 0u;  // survivor and match counts
    const int stride = len <= 16 ? 16 : (len + 15) & ~15;
    uint8_t* dst = bytes_out ? bytes_out + bucket_bytes[len] + (uint64_t)(pos - bucket_start[len]) * stride : nullptr;
    FpBuilder<VARIANT> fb;
    fb.init(P);
    uint32_t sig = 0, sigp = 0, xc = 0;  // xc: symbol codes of kXLen byte positions (exact / position path)
    for (int c = 0; c < stride; c += 16) {
        uint32_t w[4];
        const int rem = min(16, len - c);
        if (rem > 0) load_chunk(blob, beg + c, rem, w);
        else w[0] = w[1] = w[2] = w[3] = 0u;
        if (dst) *reinterpret_cast<uint4*>(dst + c) = make_uint4(w[0], w[1], w[2], w[3]);  // 16-byte aligned
#pragma unroll
        for (int t = 0; t < 16; ++t) {
            if (t < rem) {
                const uint32_t byte = (w[t >> 2] >> (8 * (t & 3))) & 0xffu;
                const int q = s_slot[byte];
                if (q >= 0) fb.add(q, c + t, len, P);
                sig |= 1u << (byte & 31);
                const int g = s_sigbit[byte];
                if (g >= 0) sigp |= 1u << g;
            }
        }
        // position codes (K2's exact / position path): every byte of a word of
        // <= kXLen bytes, else the kXLen positions floor(j * len / kXLen),
        // j = 0 .. kXLen - 1 (spread over the word; words and queries of one
        // length pick the same positions)
        if (xc_out) {
#pragma unroll
            for (int j = 0; j < kXLen; ++j) {
                const int p = len <= kXLen ? j : (j * len) / kXLen;
                if (p < len && p >= c && p < c + 16) {
                    const int o = p - c;
                    const uint32_t wv = (o >> 2) == 0 ? w[0] : (o >> 2) == 1 ? w[1] : (o >> 2) == 2 ? w[2] : w[3];
                    xc |= (uint32_t)s_xcode[(wv >> (8 * (o & 3))) & 0xffu] << (kXBits * j);
                }
            }
        }
    }
    const uint64_t fp = fb.bits;
    fp_out[pos] = fp;
    if (cmp_out) cmp_out[pos] = P.onehot ? onehot_count16(fp) : fp;
    if (sig_out) sig_out[pos] = sig;
    if (sigp_out) sigp_out[pos] = sigp;
    if (id_out) id_out[pos] = id;
    if (weight_out) weight_out[pos] = fp_gweight(fp, P);
    if (xc_out) xc_out[pos] = xc;
}

// Lengths, identity ids and the length histogram (lengths < 256 counted in
// shared memory first: a dictionary has few distinct lengths, and global
// atomics on them would serialise).  blockDim == 256.
#ifndef FPG_K2_TU  // defined once, in fpg_api.cu
__global__ void k_lengths(const uint64_t* __restrict__ offsets, uint64_t n,
                          uint16_t* __restrict__ len_out, uint32_t* __restrict__ idx_out,
                          uint32_t* __restrict__ hist, uint32_t* __restrict__ too_long) {
    __shared__ uint32_t h[256];
    h[threadIdx.x] = 0;
    __syncthreads();
    // grid-stride (a few CTAs per SM): the per-CTA flush of the shared
    // histogram to its ~L global counters happens once per CTA, not per 256 words
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i0 = (uint64_t)blockIdx.x * blockDim.x; i0 < n; i0 += stride) {
        const uint64_t i = i0 + threadIdx.x;
        uint32_t key = 0xffffffffu;  // this thread's length (none past n)
        if (i < n) {
            uint64_t len = offsets[i + 1] - offsets[i];
            if (len > (uint64_t)kMaxLen) {
                atomicAdd(too_long, 1u);
                len = kMaxLen;
            }
            len_out[i] = (uint16_t)len;
            idx_out[i] = (uint32_t)i;
            key = (uint32_t)len;
        }
        // warp-aggregated: lanes with equal lengths add once (a dictionary has
        // few distinct lengths, so per-thread shared atomics would serialise)
        const uint32_t peers = __match_any_sync(0xffffffffu, key);
        if (key != 0xffffffffu && (int)(threadIdx.x & 31) == __ffs(peers) - 1) {
            if (key < 256) atomicAdd(&h[key], (uint32_t)__popc(peers));
            else atomicAdd(&hist[key], (uint32_t)__popc(peers));
        }
    }
    __syncthreads();
    if (h[threadIdx.x]) atomicAdd(&hist[threadIdx.x], h[threadIdx.x]);
}
#endif

#ifndef FPG_K2_TU  // defined once, in fpg_api.cu
__global__ void k_scatter_prints(const uint64_t* __restrict__ fp, const uint32_t* __restrict__ ids,
                                 uint64_t n, uint64_t* __restrict__ out) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[ids[i]] = fp[i];
}
#endif

// ---------------------------------------------------------------- K4 CSR
constexpr uint32_t kSegMax = 32;  // K4 warp-sorts segments up to this size

// Match bookkeeping of one hit: per-query count (the K4 segment size).
// Called by the hit lanes of a warp (`hb` = ballot of hits, `head` = this
// lane starts a run of adjacent hit lanes with the same query, `heads` = the
// ballot of heads): one fire-and-forget reduction per run, so popular queries
// do not serialise on their counter.  Large segments are detected in K4.
__device__ __forceinline__ void count_match(uint32_t* q_matches, uint32_t qid, uint32_t hb, bool head,
                                            uint32_t heads) {
    if (!head) return;
    const int lane = threadIdx.x & 31;
    const uint32_t above = heads & (0xfffffffeu << lane);  // later heads
    const uint32_t upto = above ? ((1u << (__ffs(above) - 1)) - 1u) : 0xffffffffu;
    atomicAdd(&q_matches[qid], (uint32_t)__popc(hb & upto & (0xffffffffu << lane)));
}

// Per-warp output chunk: a warp reserves kOutChunk key slots with one atomic
// and fills them over many ballots; slots it leaves unused hold kNoKey (K4
// skips them).  Keeps the global slot counter out of the per-hit path.
constexpr uint32_t kOutChunk = 256;
constexpr unsigned long long kNoKey = ~0ull;

struct OutChunk {
    uint64_t base = ~0ull;  // first slot of the current chunk (warp-uniform)
    uint32_t fill = kOutChunk;
    uint32_t real = 0;      // hits emitted by this warp

    __device__ __forceinline__ void close(unsigned long long* out, uint64_t cap) {
        if (base == ~0ull) return;
        for (uint32_t i = fill + (threadIdx.x & 31); i < kOutChunk; i += 32)
            if (base + i < cap) out[base + i] = kNoKey;
    }
    // Warp-collective: `hit` lanes append `key`.
    __device__ __forceinline__ void emit(uint32_t hb, bool hit, unsigned long long key, unsigned long long* out,
                                         uint64_t cap, unsigned long long* slots) {
        const uint32_t h = (uint32_t)__popc(hb);
        if (fill + h > kOutChunk) {
            close(out, cap);
            unsigned long long b = 0;
            if ((threadIdx.x & 31) == 0) b = atomicAdd(slots, (unsigned long long)kOutChunk);
            base = __shfl_sync(0xffffffffu, b, 0);
            fill = 0;
        }
        if (hit) {
            const uint64_t o = base + fill + (uint32_t)__popc(hb & ((1u << (threadIdx.x & 31)) - 1u));
            if (o < cap) out[o] = key;
        }
        fill += h;
        real += h;
    }
};

// Run heads for count_match: a hit lane whose lower neighbour is not a hit
// of the same query.  Warp-collective.
__device__ __forceinline__ bool match_run_head(bool hit, uint32_t qid, uint32_t hb) {
    const int lane = threadIdx.x & 31;
    const uint32_t prev = __shfl_up_sync(0xffffffffu, qid, 1);
    return hit && (lane == 0 || !((hb >> (lane - 1)) & 1u) || prev != qid);
}

// K4 segmented (all segments <= kSegMax): keys -> their query's segment.
#ifndef FPG_K2_TU  // defined once, in fpg_api.cu
__global__ void k_seg_scatter(const unsigned long long* __restrict__ keys, const unsigned long long* __restrict__ slots,
                              const unsigned long long* __restrict__ matches, uint64_t cap,
                              const uint64_t* __restrict__ offsets_in, uint32_t* __restrict__ cursor,
                              uint32_t* __restrict__ ids, uint64_t* __restrict__ offsets_last,
                              const uint32_t* __restrict__ w_ids, uint64_t id_base) {
    const uint64_t used = *slots;
    const uint64_t n = used < cap ? used : cap;  // overflowed runs are redone by the host
    const uint64_t i0 = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int lane = threadIdx.x & 31;
    if (i0 == 0) *offsets_last = *matches;
    // warp-uniform trip count; lanes holding keys of the same query claim
    // their slots with one atomic (popular queries would serialise otherwise)
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t b = i0 - lane; b < n; b += stride) {
        const uint64_t i = b + lane;
        const unsigned long long k = i < n ? keys[i] : kNoKey;
        const uint32_t q = (uint32_t)(k >> 32);  // kNoKey -> 0xffffffff, never a query
        const uint32_t peers = __match_any_sync(0xffffffffu, q);
        if (k == kNoKey) continue;
        const int leader = __ffs(peers) - 1;
        const uint32_t cnt = (uint32_t)__popc(peers);
        uint32_t base = 0;
        if (lane == leader) base = atomicSub(&cursor[q], cnt) - cnt;
        base = __shfl_sync(peers, base, leader);
        const uint64_t pos = offsets_in[q] + base + (uint32_t)__popc(peers & ((1u << lane) - 1u));
        // K2 keys carry the word's sorted position: map it to the input-order
        // id here, where the gathers of a whole warp are in flight at once
        if (pos < cap) ids[pos] = (uint32_t)(id_base + __ldg(w_ids + (uint32_t)k));
    }
}
#endif

// One warp per query: bitonic sort of its <= 32 word ids in registers.
// Larger segments are listed for k_seg_sort_big.
#ifndef FPG_K2_TU  // defined once, in fpg_api.cu
__global__ void k_seg_sort(const uint64_t* __restrict__ offsets, uint64_t nq, uint64_t cap, uint32_t* __restrict__ ids,
                           unsigned long long* __restrict__ big_seg, uint32_t* __restrict__ big_list,
                           unsigned long long* __restrict__ n_big) {
    const uint64_t q = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (q >= nq) return;
    const uint64_t o = offsets[q];
    const uint64_t e = offsets[q + 1];
    if (e - o > kSegMax) {  // large segment: k_seg_sort_big (launched by the host after the run's sync)
        if (lane == 0 && e <= cap) {
            *big_seg = 1ull;
            big_list[atomicAdd(n_big, 1ull)] = (uint32_t)q;
        }
        return;
    }
    if (e > cap) return;  // overflowed run: the host reruns
    const int n = (int)(e - o);
    if (n <= 1) return;
    uint32_t v = lane < n ? ids[o + lane] : 0xffffffffu;
#pragma unroll
    for (int k = 2; k <= 32; k <<= 1) {
#pragma unroll
        for (int j = k >> 1; j > 0; j >>= 1) {
            const uint32_t u = __shfl_xor_sync(0xffffffffu, v, j);
            const bool up = (lane & k) == 0;
            const bool lower = (lane & j) == 0;
            v = (lower == up) ? min(v, u) : max(v, u);
        }
    }
    if (lane < n) ids[o + lane] = v;
}
#endif

// Segments of more than kSegMax ids (k_seg_sort's list), one CTA each, sorted
// in place: the ids go to B buckets of equal value range over [min, max] of
// the segment (B ~ n / 16, a power of two; tmp holds them bucket by bucket),
// then the warps sort the buckets, <= 32 ids in registers (shuffle bitonic),
// up to kBucketMax in shared memory, and write them back in bucket order.  A
// bucket above kBucketMax ids (very skewed ids) sets *overflow: the host then
// sorts every segment with CUB.
constexpr int kBigThreads = 256;
constexpr int kMaxBuckets = 2048;
constexpr int kBucketMax = 512;
#ifndef FPG_K2_TU  // defined once, in fpg_api.cu
// ascending shared-memory bitonic sort of v[0, P), P a power of two, by one warp
__device__ __forceinline__ void warp_smem_bitonic(uint32_t* v, int P, int lane) {
    for (int k = 2; k <= P; k <<= 1)
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int i = lane; i < P / 2; i += 32) {
                const int a = ((i & ~(j - 1)) << 1) | (i & (j - 1)), b = a | j;  // j is a power of two
                const uint32_t x = v[a], y = v[b];
                if ((x > y) == ((a & k) == 0)) {
                    v[a] = y;
                    v[b] = x;
                }
            }
            __syncwarp();
        }
}
// ascending bitonic sort of one value per lane (lanes past the data hold ~0)
__device__ __forceinline__ uint32_t warp_reg_bitonic(uint32_t v, int lane) {
#pragma unroll
    for (int k = 2; k <= 32; k <<= 1)
#pragma unroll
        for (int j = k >> 1; j > 0; j >>= 1) {
            const uint32_t u = __shfl_xor_sync(0xffffffffu, v, j);
            const bool up = (lane & k) == 0, lower = (lane & j) == 0;
            v = (lower == up) ? min(v, u) : max(v, u);
        }
    return v;
}

__global__ void __launch_bounds__(kBigThreads) k_seg_sort_big(const uint64_t* __restrict__ offsets,
                                                              const uint32_t* __restrict__ big_list, uint64_t n_big,
                                                              uint32_t* __restrict__ ids, uint32_t* __restrict__ tmp,
                                                              unsigned long long* __restrict__ overflow) {
    constexpr int NW = kBigThreads / 32;
    __shared__ uint32_t s_cnt[kMaxBuckets], s_cur[kMaxBuckets];
    __shared__ uint32_t s_wv[NW][kBucketMax];
    __shared__ uint32_t s_lo, s_hi, s_over;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (uint64_t bi = blockIdx.x; bi < n_big; bi += gridDim.x) {
        const uint32_t q = big_list[bi];
        const uint64_t o = offsets[q];
        const int n = (int)(offsets[q + 1] - o);
        uint32_t* seg = ids + o;
        int B = 32;
        while (B < n / 16 && B < kMaxBuckets) B <<= 1;
        if (tid == 0) {
            s_lo = 0xffffffffu;
            s_hi = 0u;
            s_over = 0u;
        }
        for (int i = tid; i < B; i += kBigThreads) s_cnt[i] = 0u;
        uint32_t lo = 0xffffffffu, hi = 0u;
        for (int i = tid; i < n; i += kBigThreads) {
            const uint32_t v = seg[i];
            lo = min(lo, v);
            hi = max(hi, v);
        }
        lo = __reduce_min_sync(0xffffffffu, lo);
        hi = __reduce_max_sync(0xffffffffu, hi);
        __syncthreads();
        if (lane == 0) {
            atomicMin(&s_lo, lo);
            atomicMax(&s_hi, hi);
        }
        __syncthreads();
        lo = s_lo;
        const uint64_t span = (uint64_t)s_hi - lo + 1;
        // bucket = floor((v - lo) * B / span) without a 64-bit division per id
        // (which cost more than the rest of the kernel): a multiply by
        // floor(B * 2^32 / span) and a shift give the quotient or one less,
        // and one more multiply decides which
        const uint64_t scale = ((uint64_t)B << 32) / span;
        auto bucket = [&](uint32_t v) {
            const uint64_t d = v - lo;
            uint32_t b = (uint32_t)((d * scale) >> 32);
            if ((uint64_t)(b + 1u) * span <= d * (uint64_t)B) ++b;
            return (int)b;
        };
        for (int i = tid; i < n; i += kBigThreads) atomicAdd(&s_cnt[bucket(seg[i])], 1u);
        __syncthreads();
        // exclusive scan of the bucket counts (one warp)
        if (warp == 0) {
            uint32_t run = 0;
            for (int b0 = 0; b0 < B; b0 += 32) {
                const uint32_t c = s_cnt[b0 + lane];
                if (c > (uint32_t)kBucketMax) s_over = 1u;
                uint32_t incl = c;
#pragma unroll
                for (int d = 1; d < 32; d <<= 1) {
                    const uint32_t v = __shfl_up_sync(0xffffffffu, incl, d);
                    if (lane >= d) incl += v;
                }
                s_cur[b0 + lane] = run + incl - c;
                run += __shfl_sync(0xffffffffu, incl, 31);
            }
        }
        __syncthreads();
        if (s_over) {  // left to the host's CUB fallback
            if (tid == 0) *overflow = 1ull;
            __syncthreads();
            continue;
        }
        for (int i = tid; i < n; i += kBigThreads) {
            const uint32_t v = seg[i];
            tmp[o + atomicAdd(&s_cur[bucket(v)], 1u)] = v;
        }
        __syncthreads();
        // s_cur[b] is now the end of bucket b; its start is s_cur[b] - s_cnt[b]
        for (int b = warp; b < B; b += NW) {
            const int c = (int)s_cnt[b];
            if (!c) continue;
            const uint32_t st = s_cur[b] - (uint32_t)c;
            if (c <= 32) {
                uint32_t v = lane < c ? tmp[o + st + lane] : 0xffffffffu;
                v = warp_reg_bitonic(v, lane);
                if (lane < c) seg[st + lane] = v;
            } else {
                int P = 64;
                while (P < c) P <<= 1;
                uint32_t* wv = s_wv[warp];
                for (int i = lane; i < P; i += 32) wv[i] = i < c ? tmp[o + st + i] : 0xffffffffu;
                __syncwarp();
                warp_smem_bitonic(wv, P, lane);
                for (int i = lane; i < c; i += 32) seg[st + i] = wv[i];
                __syncwarp();
            }
        }
        __syncthreads();
    }
}
#endif

// ---------------------------------------------------------------- QueryStats by fingerprint histogram
// W = 16 dictionaries: QueryStats::verified (dictionary.hpp:102-110: the
// words that pass the length test and the fingerprint test F_D <= 2k) does not
// need the pair scan.  F_D counts the fields whose bits differ
// (ComparisonTables, fingerprint.hpp:171-214), so the fingerprints within
// F_D <= 2k of a query's are fp ^ d for the XOR masks d that touch at most 2k
// fields (137 masks for 16 one-bit fields at k = 1, 277 for count-16 b = 2,
// 562 for position-16 p = 3; the host lists them, 0 first), and
//     verified(q) = sum over compatible lengths L, masks d of H_L[fp(q) ^ d]
// with H_L the histogram of the fingerprints of the words of length L.  K2
// then runs without its survivor counters.
//
// k_fp_hist: H[slot(L)][fp] over the sorted dictionary (slot nh = all lengths).
#ifndef FPG_K2_TU  // defined once, in fpg_api.cu
__global__ void k_fp_hist(const uint64_t* __restrict__ fp, uint64_t n, const uint32_t* __restrict__ slot_first,
                          int nh, uint32_t* __restrict__ hist) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    int lo = 0, hi = nh;  // largest slot with slot_first[slot] <= i
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (slot_first[mid] <= i) lo = mid;
        else hi = mid;
    }
    const uint32_t f = (uint32_t)fp[i] & 0xffffu;
    atomicAdd(&hist[(uint64_t)lo * 65536u + f], 1u);
    atomicAdd(&hist[(uint64_t)nh * 65536u + f], 1u);
}

// One warp per (sorted) query.  span: compatible lengths are m - span .. m +
// span; all_lengths: every word is length-compatible (Levenshtein without the
// length prefilter, dictionary.hpp:94-101).
__global__ void __launch_bounds__(256) k_fp_stats(const uint64_t* __restrict__ q_fp, const uint16_t* __restrict__ q_len,
                                                  const uint32_t* __restrict__ q_ids, uint64_t nq,
                                                  const uint32_t* __restrict__ hist, const int32_t* __restrict__ hslot,
                                                  int nh, int max_len, const uint16_t* __restrict__ deltas, int nd,
                                                  int span, int all_lengths, uint32_t* __restrict__ q_survivors,
                                                  unsigned long long* __restrict__ survivors_total) {
    const int lane = threadIdx.x & 31;
    const uint64_t warps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    unsigned long long warp_sum = 0;
    for (uint64_t q = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; q < nq; q += warps) {
        const uint32_t f = (uint32_t)q_fp[q] & 0xffffu;
        const int m = (int)q_len[q];
        const uint32_t* h[3] = {nullptr, nullptr, nullptr};
        if (all_lengths) {
            h[0] = hist + (uint64_t)nh * 65536u;
        } else {
            for (int t = 0; t <= 2 * span; ++t) {
                const int L = m - span + t;
                const int sl = (L >= 0 && L <= max_len) ? hslot[L] : -1;
                if (sl >= 0) h[t] = hist + (uint64_t)sl * 65536u;
            }
        }
        uint32_t c = 0;
        for (int i = lane; i < nd; i += 32) {
            const uint32_t g = f ^ (uint32_t)deltas[i];
#pragma unroll
            for (int t = 0; t < 3; ++t)
                if (h[t]) c += __ldg(h[t] + g);
        }
        c = __reduce_add_sync(0xffffffffu, c);
        if (lane == 0) {
            q_survivors[q_ids[q]] = c;
            warp_sum += c;
        }
    }
    if (lane == 0 && warp_sum) atomicAdd(survivors_total, warp_sum);
}
#endif

// ---------------------------------------------------------------- CSR merge
// Shards own ascending, contiguous input-order id ranges, so the global
// (query asc, word asc) CSR is each query's part rows concatenated in part
// order: a gather, not a sort.
constexpr int kMaxMergeParts = 16;
struct MergeParts {
    int n;
    const uint64_t* off[kMaxMergeParts];  // nq + 1 offsets per part
    const uint32_t* ids[kMaxMergeParts];
};

// cnt[q] = sum over parts of row q's length, cnt[nq] = 0 (the scan's total).
#ifndef FPG_K2_TU  // defined once, in fpg_api.cu
__global__ void k_merge_counts(const __grid_constant__ MergeParts mp, uint64_t nq, uint64_t* __restrict__ cnt) {
    for (uint64_t q = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; q <= nq; q += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t c = 0;
        if (q < nq)
            for (int p = 0; p < mp.n; ++p) c += __ldg(mp.off[p] + q + 1) - __ldg(mp.off[p] + q);
        cnt[q] = c;
    }
}
#endif

// One warp per query: its part rows, in part order, to the merged row.
#ifndef FPG_K2_TU  // defined once, in fpg_api.cu
__global__ void k_merge_rows(const __grid_constant__ MergeParts mp, uint64_t nq, const uint64_t* __restrict__ out_off,
                             uint32_t* __restrict__ out_ids) {
    const int lane = threadIdx.x & 31;
    const uint64_t warps = (uint64_t)gridDim.x * blockDim.x / 32;
    for (uint64_t q = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) / 32; q < nq; q += warps) {
        uint64_t at = out_off[q];
        for (int p = 0; p < mp.n; ++p) {
            const uint64_t a = __ldg(mp.off[p] + q), b = __ldg(mp.off[p] + q + 1);
            for (uint64_t i = a + lane; i < b; i += 32) out_ids[at + (i - a)] = __ldg(mp.ids[p] + i);
            at += b - a;
        }
    }
}
#endif

}  // namespace fpg

#include "fpg_scan.cuh"
#include "fpg_verify.cuh"
#include "fpg_slice.cuh"
