// fpg_scan.cuh -- K2: the fused filter + k<=1 verify scan (sm_100a).
//
// One CTA = 8 warps = one tile: up to 2048 words of one dictionary length
// bucket (8 per lane, comparison words in registers) x up to 256 queries of
// one query length bucket (comparison words in shared memory, read as warp
// broadcasts).  For every (query, word) pair the reference's fingerprint test
// (dictionary.hpp:102-106: ceil_half(F_D) > k, i.e. F_D > 2k) runs as one
// XOR + POPC (+ a compile-time field fold for count / position layouts,
// ComparisonTables fingerprint.hpp:180-194).  Survivors are appended without
// any warp vote to a lane-private queue in shared memory (slot-major
// [slot][lane] layout: conflict-free), and when any lane's queue is nearly
// full the warp verifies all queued candidates slot by slot with register-
// resident byte compares (hamming_bounded / levenshtein_bounded at k<=1,
// edit_distance.hpp:18-64).  Matches (rare) leave through a warp-aggregated
// atomic append; per-query survivor counts (QueryStats::verified) come from
// one REDUX per warp and query.
#pragma once

#include <cstdint>
#include <type_traits>

namespace fpg {

enum DistKind : int { kPopc = 0, kFold2 = 1, kFold4 = 2, kPos3 = 3, kGeneric = 4 };

template <typename T>
__device__ __forceinline__ int popcnt(T x) {
    if constexpr (sizeof(T) == 8) return __popcll(x);
    else return __popc(x);
}

// F_D on the comparison words' xor.  kPopc covers occurrence, halved and the
// one-hot count-16 form (whose popcount is twice F_D; the threshold is doubled
// on the host instead).
template <int KIND, typename T>
__device__ __forceinline__ int distance_of(T x, T mf, T ms, int fold) {
    if constexpr (KIND == kPopc) {
        return popcnt(x);
    } else if constexpr (KIND == kFold2) {
        return popcnt((x | (x >> 1)) & mf);
    } else if constexpr (KIND == kFold4) {
        return popcnt((x | (x >> 1) | (x >> 2) | (x >> 3)) & mf);
    } else if constexpr (KIND == kPos3) {
        return popcnt(((x | (x >> 1) | (x >> 2)) & mf) | (x & ms));
    } else {
        T f = x;
        for (int j = 1; j < fold; ++j) f |= x >> j;
        return popcnt((f & mf) | (x & ms));
    }
}

__device__ __forceinline__ uint32_t ld32(const uint8_t* base, int chunk, int stride) {
    return (4 * chunk < stride) ? __ldg(reinterpret_cast<const uint32_t*>(base) + chunk) : 0u;
}

// k<=1 verification of zero-padded byte strings, any length (global loads).
// Semantics of hamming_bounded / levenshtein_bounded (edit_distance.hpp:18-64):
//   equal lengths: distance <= 1  <=>  first mismatching byte == last one;
//   lengths differ by one (long s, short t): t is s with one byte deleted  <=>
//   (last mismatch of t vs s shifted left by one byte) < (first mismatch of t vs s).
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

// Same test with both strings already in registers (NW 32-bit words, zero
// padded, NW*4 >= max(m, n)).
template <int NW>
__device__ __forceinline__ bool verify_regs(const uint32_t (&q)[NW], const uint32_t (&w)[NW], int m,
                                            int n, int k) {
    if (m == n) {
        int fi = NW, li = -1;
        uint32_t fx = 0, lx = 0;
#pragma unroll
        for (int i = NW - 1; i >= 0; --i) {
            const uint32_t x = q[i] ^ w[i];
            if (x) { fi = i; fx = x; }
        }
        if (fi == NW) return true;
        if (k == 0) return false;
#pragma unroll
        for (int i = 0; i < NW; ++i) {
            const uint32_t x = q[i] ^ w[i];
            if (x) { li = i; lx = x; }
        }
        return fi == li && ((__ffs(fx) - 1) >> 3) == ((31 - __clz(lx)) >> 3);
    }
    if (k == 0) return false;
    const bool wl = n > m;  // tile-uniform
    int fi = NW, li = -1;
    uint32_t fx = 0, lx = 0;
#pragma unroll
    for (int i = NW - 1; i >= 0; --i) {
        const uint32_t a = q[i] ^ w[i];
        if (a) { fi = i; fx = a; }
    }
    if (fi == NW) return true;  // shorter is a prefix of longer (and the extra byte is 0)
#pragma unroll
    for (int i = 0; i < NW; ++i) {
        const uint32_t s0 = wl ? w[i] : q[i];
        const uint32_t s1 = (i + 1 < NW) ? (wl ? w[i + 1] : q[i + 1]) : 0u;
        const uint32_t t0 = wl ? q[i] : w[i];
        const uint32_t b = t0 ^ __funnelshift_r(s0, s1, 8);
        if (b) { li = i; lx = b; }
    }
    if (li < 0) return true;
    const int fa = 4 * fi + ((__ffs(fx) - 1) >> 3);
    const int lb = 4 * li + ((31 - __clz(lx)) >> 3);
    return lb < fa;
}

template <int NW>
__device__ __forceinline__ void load_padded(const uint8_t* p, int stride, uint32_t (&r)[NW]) {
    const uint4 a = __ldg(reinterpret_cast<const uint4*>(p));
    r[0] = a.x; r[1] = a.y; r[2] = a.z; r[3] = a.w;
    if constexpr (NW == 8) {
        uint4 b = make_uint4(0, 0, 0, 0);
        if (stride > 16) b = __ldg(reinterpret_cast<const uint4*>(p) + 1);
        r[4] = b.x; r[5] = b.y; r[6] = b.z; r[7] = b.w;
    }
}

constexpr int kScanThreads = 256;
constexpr int kScanWarps = kScanThreads / 32;
constexpr int kWordsPerLane = 8;                                   // R
constexpr int kTileWords = kScanThreads * kWordsPerLane;           // 2048
constexpr int kTileQueries = 256;
constexpr int kLaneCap = 24;                                       // queue slots per lane

// 32-bit shared-window addressing (keeps generic->shared conversions out of loops).
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void sts32(uint32_t a, uint32_t v) {
    asm volatile("st.shared.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t lds32(uint32_t a) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
    return v;
}
template <typename T>
__device__ __forceinline__ T lds_t(uint32_t a) {
    if constexpr (sizeof(T) == 8) {
        uint64_t v;
        asm volatile("ld.shared.u64 %0, [%1];" : "=l"(v) : "r"(a) : "memory");
        return v;
    } else {
        return lds32(a);
    }
}

// popc(x) <= 2 without the XU pipe (clear the lowest set bit twice).
__device__ __forceinline__ bool popc_le2(uint32_t x) {
    const uint32_t y = x & (x - 1);
    return (y & (y - 1)) == 0;
}

// Per-tile state of one warp (all members live in registers once inlined).
template <int KIND, typename T, bool STATS>
struct TileScan {
    const ScanParams& P;
    const Tile& tl;
    const uint8_t* qbytes;
    const uint8_t* wbytes;
    int m, n, qs, ws, vclass, tid, lane;
    uint32_t a_queue;    // shared address of this lane's queue slot 0 (slot s at + 128 s)
    uint32_t a_qlimit;   // flush once the next push could pass the last slot
    uint32_t a_qsig;
    uint32_t qp;

    __device__ __forceinline__ bool verify_bytes(uint32_t j, uint32_t widx) const {
        const uint8_t* qb = qbytes + (uint64_t)j * qs;
        const uint8_t* wb = wbytes + (uint64_t)widx * ws;
        if (vclass == 1) {
            uint32_t a[4], b[4];
            load_padded<4>(qb, qs, a);
            load_padded<4>(wb, ws, b);
            return verify_regs<4>(a, b, m, n, P.k);
        }
        if (vclass == 2) {
            uint32_t a[8], b[8];
            load_padded<8>(qb, qs, a);
            load_padded<8>(wb, ws, b);
            return verify_regs<8>(a, b, m, n, P.k);
        }
        return verify_pair(qb, m, qs, wb, n, ws, P.k);
    }

    // Verifies every queued entry of the warp by byte compares.  Entry =
    // (j << 16) | mask(j+1) << 8 | mask(j): pairs of queries j, j+1 with this
    // lane's 8 words that passed both the fingerprint and the signature test.
    __device__ __forceinline__ void flush() {
        __syncwarp();
        const uint32_t lt_mask = (1u << lane) - 1u;
        const int cnt = (int)((qp - a_queue) >> 7);
        const int maxc = (int)__reduce_max_sync(0xffffffffu, (unsigned)cnt);
        for (int s = 0; s < maxc; ++s) {
            uint32_t e = 0;
            if (s < cnt) e = lds32(a_queue + 128u * s);
            const uint32_t j0 = e >> 16;
            uint32_t keep = e & 0xffffu;
            while (__any_sync(0xffffffffu, keep != 0)) {
                bool hit = false;
                uint32_t j = 0, widx = 0;
                if (keep) {
                    const int b = 31 - __clz(keep);
                    keep ^= 1u << b;
                    j = j0 + (b >> 3);
                    widx = (uint32_t)((b & 7) * kScanThreads + tid);
                    hit = verify_bytes(j, widx);
                }
                const uint32_t hb = __ballot_sync(0xffffffffu, hit);
                if (hb) {
                    unsigned long long slot = 0;
                    if (lane == 0) slot = atomicAdd(P.out_count, (unsigned long long)__popc(hb));
                    slot = __shfl_sync(0xffffffffu, slot, 0);
                    if (hit) {
                        const uint64_t o = slot + __popc(hb & lt_mask);
                        if (o < P.out_cap) {
                            const uint64_t qid = P.q_ids[tl.q_begin + j];
                            const uint64_t wid = P.id_base + P.w_ids[tl.w_begin + widx];
                            P.out[o] = (qid << 32) | wid;
                        }
                    }
                }
            }
        }
        __syncwarp();
        qp = a_queue;
    }

    // Filter loop over the tile's queries, two per iteration.  Per pair: the
    // reference fingerprint test (counted for QueryStats) and the exact
    // occurrence-signature test; pairs passing both are queued.  The
    // signature popcount runs on the XU pipe for words 0..4 and as ALU
    // bit-clears for words 5..7, balancing the two pipes.  FULL: all 8 words
    // of every lane are valid (all but each bucket's last tile).  Returns the
    // warp's fingerprint-survivor count (STATS only).
    template <bool FULL>
    __device__ __forceinline__ unsigned scan(uint32_t a_q, const T (&wc)[kWordsPerLane],
                                             const uint32_t (&wg)[kWordsPerLane],
                                             const bool (&wv)[kWordsPerLane], uint32_t a_wsurv) {
        const T mf = (T)P.mask_fold, ms = (T)P.mask_single;
        const int thr = P.thr;
        unsigned total = 0;
        for (uint32_t j = 0; j < tl.q_count; j += 2) {
            const bool two = j + 1 < tl.q_count;
            const uint32_t j1 = two ? j + 1 : j;
            const T q0 = lds_t<T>(a_q + (uint32_t)sizeof(T) * j);
            const T q1 = lds_t<T>(a_q + (uint32_t)sizeof(T) * j1);
            const uint32_t g0 = lds32(a_qsig + 4u * j);
            const uint32_t g1 = lds32(a_qsig + 4u * j1);
            uint32_t mfp = 0, mboth = 0;
#pragma unroll
            for (int r = 0; r < kWordsPerLane; ++r) {
                bool f0 = distance_of<KIND, T>(q0 ^ wc[r], mf, ms, P.fold) <= thr;
                bool f1 = distance_of<KIND, T>(q1 ^ wc[r], mf, ms, P.fold) <= thr;
                if constexpr (!FULL) { f0 &= wv[r]; f1 &= wv[r]; }
                bool s0, s1;
                if (r < 5) {
                    s0 = __popc(g0 ^ wg[r]) <= 2;
                    s1 = __popc(g1 ^ wg[r]) <= 2;
                } else {
                    s0 = popc_le2(g0 ^ wg[r]);
                    s1 = popc_le2(g1 ^ wg[r]);
                }
                mfp |= (f0 ? (1u << r) : 0u) | (f1 ? (0x100u << r) : 0u);
                mboth |= ((f0 & s0) ? (1u << r) : 0u) | ((f1 & s1) ? (0x100u << r) : 0u);
            }
            if (!two) { mfp &= 0xffu; mboth &= 0xffu; }
            sts32(qp, (j << 16) | mboth);  // unconditional: the slot is free until qp moves
            qp += mboth ? 128u : 0u;
            if constexpr (STATS) {
                const unsigned c = __reduce_add_sync(0xffffffffu, (unsigned)(__popc(mfp & 0xffu) | (__popc(mfp >> 8) << 16)));
                if (lane == 0) {
                    sts32(a_wsurv + 4u * j, c & 0xffffu);
                    if (two) sts32(a_wsurv + 4u * j1, c >> 16);
                }
                total += (c & 0xffffu) + (c >> 16);
            }
            if (__any_sync(0xffffffffu, qp > a_qlimit)) flush();
        }
        flush();
        return total;
    }
};

template <int KIND, int W, bool STATS>
__global__ void __launch_bounds__(kScanThreads, 4) k_scan(const Tile* __restrict__ tiles, uint32_t ntiles,
                                                          const __grid_constant__ ScanParams P) {
    using T = typename std::conditional<(W <= 32), uint32_t, uint64_t>::type;
    __shared__ T s_q[kTileQueries];
    __shared__ uint32_t s_qsig[kTileQueries];
    __shared__ uint32_t s_wsurv[STATS ? kScanWarps : 1][STATS ? kTileQueries : 1];
    __shared__ uint32_t s_queue[kScanWarps * kLaneCap * 32];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    // lane-private queue, slot-major: slot s of this lane at word (warp*cap + s)*32 + lane
    const uint32_t a_queue = smem_u32(s_queue) + 4u * (uint32_t)(warp * kLaneCap * 32 + lane);
    const uint32_t a_q = smem_u32(s_q), a_qsig = smem_u32(s_qsig);
    const uint32_t a_wsurv = smem_u32(s_wsurv[STATS ? warp : 0]);
    unsigned long long surv_warp = 0;  // lane 0's copy is the warp total (STATS)

    for (uint32_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const Tile tl = tiles[t];
        __syncthreads();  // previous tile's shared state fully consumed
        for (uint32_t i = tid; i < tl.q_count; i += kScanThreads) {
            s_q[i] = (T)P.q_fp[tl.q_begin + i];
            s_qsig[i] = P.q_sig[tl.q_begin + i];
        }
        T wc[kWordsPerLane];
        uint32_t wg[kWordsPerLane];
        bool wv[kWordsPerLane];
#pragma unroll
        for (int r = 0; r < kWordsPerLane; ++r) {
            const uint32_t widx = r * kScanThreads + tid;
            wv[r] = widx < tl.w_count;
            wc[r] = wv[r] ? (T)P.w_fp[tl.w_begin + widx] : (T)0;
            wg[r] = wv[r] ? P.w_sig[tl.w_begin + widx] : 0u;
        }
        __syncthreads();

        if (!tl.count_only) {
            TileScan<KIND, T, STATS> ts{P, tl, P.q_bytes + tl.q_bytes, P.w_bytes + tl.w_bytes,
                                        tl.q_len, tl.w_len, tl.q_stride, tl.w_stride,
                                        (tl.q_len <= 16 && tl.w_len <= 16) ? 1 : (tl.q_len <= 32 && tl.w_len <= 32) ? 2 : 0,
                                        tid, lane, a_queue, a_queue + 128u * (kLaneCap - 1), a_qsig, a_queue};
            surv_warp += (tl.w_count == kTileWords) ? ts.template scan<true>(a_q, wc, wg, wv, a_wsurv)
                                                    : ts.template scan<false>(a_q, wc, wg, wv, a_wsurv);
        } else if constexpr (STATS) {
            // incompatible lengths with the length prefilter off: the reference
            // still runs the fingerprint test (dictionary.hpp:102-106) and
            // counts survivors as verified; the verifier rejects them by length.
            const T mf = (T)P.mask_fold, ms = (T)P.mask_single;
            for (uint32_t j = 0; j < tl.q_count; ++j) {
                const T qc = s_q[j];
                unsigned c = 0;
#pragma unroll
                for (int r = 0; r < kWordsPerLane; ++r)
                    c += ((distance_of<KIND, T>(qc ^ wc[r], mf, ms, P.fold) <= P.thr) & wv[r]) ? 1u : 0u;
                c = __reduce_add_sync(0xffffffffu, c);
                if (lane == 0) s_wsurv[warp][j] = c;
                surv_warp += c;
            }
        }
        if constexpr (STATS) {
            __syncthreads();
            for (uint32_t i = tid; i < tl.q_count; i += kScanThreads) {
                uint32_t v = 0;
#pragma unroll
                for (int w = 0; w < kScanWarps; ++w) v += s_wsurv[w][i];
                if (v) atomicAdd(&P.q_survivors[P.q_ids[tl.q_begin + i]], v);
            }
        }
    }
    // run total of fingerprint survivors (reported), one atomic per warp
    if (STATS && lane == 0 && surv_warp) atomicAdd(P.survivors_total, surv_warp);
}

}  // namespace fpg
