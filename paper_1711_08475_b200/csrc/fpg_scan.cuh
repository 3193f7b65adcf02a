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

// k >= 2 verification from global memory (zero-padded strings).
constexpr int kMaxK = 8;  // largest k the GPU scan accepts

// hamming_bounded (edit_distance.hpp:18-27) as a test: equal lengths, at most
// k mismatching bytes.  Padding is zero on both sides, so whole 4-byte words
// compare; bytes that differ are counted per word.
__device__ __forceinline__ bool hamming_le(const uint8_t* a, const uint8_t* b, int n, int k) {
    int mism = 0;
    for (int c = 0; c < n; c += 4) {
        uint32_t x = __ldg(reinterpret_cast<const uint32_t*>(a + c)) ^ __ldg(reinterpret_cast<const uint32_t*>(b + c));
        x = (x | (x >> 4)) & 0x0f0f0f0fu;
        x = (x | (x >> 2)) & 0x03030303u;
        x = (x | (x >> 1)) & 0x01010101u;
        mism += __popc(x);
        if (mism > k) return false;
    }
    return true;
}

// levenshtein_bounded (edit_distance.hpp:31-64) as a test: the 2k+1-wide
// band of the DP, cell (i, j) at band index t = j - i + k, early exit when a
// row's minimum exceeds k.
static __device__ __noinline__ bool levenshtein_le(const uint8_t* s1, int m, const uint8_t* s2, int n, int k) {
    if (m > n) {
        const uint8_t* ts = s1; s1 = s2; s2 = ts;
        const int tn = m; m = n; n = tn;
    }
    if (n - m > k) return false;
    const int inf = k + 1, w = 2 * k + 1;
    int prev[2 * kMaxK + 1], cur[2 * kMaxK + 1];
    for (int t = 0; t < w; ++t) {  // row 0: D[0][j] = j
        const int j = t - k;
        prev[t] = (j < 0 || j > n || j > k) ? inf : j;
    }
    for (int i = 1; i <= m; ++i) {
        const uint8_t a = __ldg(s1 + i - 1);
        int best = inf;
        for (int t = 0; t < w; ++t) {
            const int j = i - k + t;
            int v = inf;
            if (j == 0) {
                v = i < inf ? i : inf;
            } else if (j > 0 && j <= n) {
                v = prev[t] + (a != __ldg(s2 + j - 1));               // substitution / match
                if (t + 1 < w) v = min(v, prev[t + 1] + 1);           // deletion
                if (t > 0) v = min(v, cur[t - 1] + 1);                // insertion
                v = min(v, inf);
            }
            cur[t] = v;
            best = min(best, v);
        }
        if (best > k) return false;
        for (int t = 0; t < w; ++t) prev[t] = cur[t];
    }
    return prev[n - m + k] <= k;
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
constexpr int kLaneCap = 16;                                       // queue slots per lane

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

// Pass flags of 4 fingerprint distances at once: d_t (<= 64) packed into byte t,
// byte + (127 - thr) carries into bit 7 exactly when d_t > thr (no byte overflows
// since 64 + 127 < 256).  Returns bit 8t+7 set iff d_t <= thr.
__device__ __forceinline__ uint32_t pass_flags4(uint32_t d0, uint32_t d1, uint32_t d2, uint32_t d3,
                                                uint32_t bias) {
    const uint32_t packed = d0 + d1 * 0x100u + d2 * 0x10000u + d3 * 0x1000000u;
    return ~(packed + bias) & 0x80808080u;
}

// Queue entry / mask layout.  An iteration compares queries j, j+1 (qi = 0, 1)
// with the lane's words r = 4h + t (h, t in 0..3 x 0..1).  Flag register
// k = 2 qi + h holds word t at bit 8t+7; the four registers are merged as
// f0 | f1 >> 1 | f2 >> 2 | f3 >> 3 (bit 8t+7-k) and compressed to 16 bits:
// mask bit i <-> t = i >> 2, k = 3 - (i & 3).
__device__ __forceinline__ uint32_t merge_flags(uint32_t f0, uint32_t f1, uint32_t f2, uint32_t f3) {
    return f0 | (f1 >> 1) | (f2 >> 2) | (f3 >> 3);
}
__device__ __forceinline__ uint32_t compress16(uint32_t m) {  // bits 4..7 of each byte -> 16 bits
    const uint32_t z = (m >> 4) | (m >> 8);
    return __byte_perm(z, 0, 0x4420);                          // bytes 0, 2 of z
}
__device__ __forceinline__ void decode_bit(int i, uint32_t& qi, uint32_t& r) {
    const int t = i >> 2, k = 3 - (i & 3);
    qi = (uint32_t)(k >> 1);
    r = (uint32_t)(4 * (k & 1) + t);
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
    uint32_t a_qlimit;   // flush once qp passes the last slot
    uint32_t a_qsig;
    uint32_t qp;
    OutChunk& oc;

    __device__ __forceinline__ bool verify_bytes(uint32_t j, uint32_t widx) const {
        const uint8_t* qb = qbytes + (uint64_t)j * qs;
        const uint8_t* wb = wbytes + (uint64_t)widx * ws;
        if (P.k >= 2) return m == n ? hamming_le(qb, wb, m, P.k) || (P.lev && levenshtein_le(qb, m, wb, n, P.k))
                                    : P.lev && levenshtein_le(qb, m, wb, n, P.k);
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

    // Byte-verifies every queued entry of the warp.  Entry = (j << 16) | m16:
    // the pairs of queries j, j+1 with this lane's words that passed both the
    // fingerprint and the signature test (rare: each lane walks its own bits).
    __device__ __forceinline__ void flush() {
        __syncwarp();
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
                    const int i = 31 - __clz(keep);
                    keep ^= 1u << i;
                    uint32_t qi, r;
                    decode_bit(i, qi, r);
                    j = j0 + qi;
                    widx = r * kScanThreads + (uint32_t)tid;
                    hit = verify_bytes(j, widx);
                }
                const uint32_t hb = __ballot_sync(0xffffffffu, hit);
                if (hb) {
                    const uint32_t qid = hit ? P.q_ids[tl.q_begin + j] : 0xffffffffu;
                    const bool head = match_run_head(hit, qid, hb);
                    const uint32_t heads = __ballot_sync(0xffffffffu, head);
                    const uint64_t wid = hit ? (uint64_t)(tl.w_begin + widx) : 0;  // sorted position (K4 maps it)
                    oc.emit(hb, hit, ((uint64_t)qid << 32) | wid, P.out, P.out_cap, P.out_count);
                    if (hit) count_match(P.q_matches, qid, hb, head, heads);
                }
            }
        }
        __syncwarp();
        qp = a_queue;
    }

    // Filter loop over the tile's queries, two per iteration (16 pairs per
    // lane).  Per pair: the reference fingerprint test (its survivors are the
    // QueryStats::verified count) and the exact occurrence-signature test
    // (popc(sig_q ^ sig_w) <= 2); both results as packed-byte flags, 4 pairs
    // per register.  Signature popcounts of words 0..3 run on the XU pipe,
    // words 4..7 as ALU bit-clears, balancing the two pipes.  Pairs passing
    // both tests are queued as one (j, 16-bit mask) entry.  vmask clears
    // invalid words (a bucket's last tile).  Returns the warp's fingerprint
    // survivor count (STATS only).
    __device__ __forceinline__ unsigned scan(uint32_t a_q, const T (&wc)[kWordsPerLane],
                                             const uint32_t (&wg)[kWordsPerLane], uint32_t vmask,
                                             uint32_t a_wsurv) {
        const T mf = (T)P.mask_fold, ms = (T)P.mask_single;
        const uint32_t bias = (uint32_t)(127 - min(P.thr, 127)) * 0x01010101u;
        constexpr uint32_t sbias = 125u * 0x01010101u;  // signature: popc <= 2 passes
        unsigned total = 0;
        for (uint32_t j = 0; j < tl.q_count; j += 2) {
            const bool two = j + 1 < tl.q_count;
            const uint32_t j1 = two ? j + 1 : j;
            const T q0 = lds_t<T>(a_q + (uint32_t)sizeof(T) * j);
            const T q1 = lds_t<T>(a_q + (uint32_t)sizeof(T) * j1);
            const uint32_t g0 = P.sig_on ? lds32(a_qsig + 4u * j) : 0u;
            const uint32_t g1 = P.sig_on ? lds32(a_qsig + 4u * j1) : 0u;
            uint32_t d[2][kWordsPerLane], s[2][kWordsPerLane];
#pragma unroll
            for (int r = 0; r < kWordsPerLane; ++r) {
                d[0][r] = (uint32_t)distance_of<KIND, T>(q0 ^ wc[r], mf, ms, P.fold);
                d[1][r] = (uint32_t)distance_of<KIND, T>(q1 ^ wc[r], mf, ms, P.fold);
                if (r < 4) {
                    s[0][r] = (uint32_t)__popc(g0 ^ wg[r]);
                    s[1][r] = (uint32_t)__popc(g1 ^ wg[r]);
                } else {
                    s[0][r] = popc_le2(g0 ^ wg[r]) ? 0u : 3u;
                    s[1][r] = popc_le2(g1 ^ wg[r]) ? 0u : 3u;
                }
            }
            const uint32_t f0 = pass_flags4(d[0][0], d[0][1], d[0][2], d[0][3], bias);
            const uint32_t f1 = pass_flags4(d[0][4], d[0][5], d[0][6], d[0][7], bias);
            const uint32_t f2 = pass_flags4(d[1][0], d[1][1], d[1][2], d[1][3], bias);
            const uint32_t f3 = pass_flags4(d[1][4], d[1][5], d[1][6], d[1][7], bias);
            const uint32_t t0 = pass_flags4(s[0][0], s[0][1], s[0][2], s[0][3], sbias);
            const uint32_t t1 = pass_flags4(s[0][4], s[0][5], s[0][6], s[0][7], sbias);
            const uint32_t t2 = pass_flags4(s[1][0], s[1][1], s[1][2], s[1][3], sbias);
            const uint32_t t3 = pass_flags4(s[1][4], s[1][5], s[1][6], s[1][7], sbias);
            uint32_t vm = vmask;
            if (!two) vm &= 0xC0C0C0C0u;  // keep qi = 0 (k = 0, 1 -> bits 7, 6)
            const uint32_t both = merge_flags(f0 & t0, f1 & t1, f2 & t2, f3 & t3) & vm;
            sts32(qp, __byte_perm(compress16(both), j, 0x5410));  // unconditional: slot free until qp moves
            qp += both ? 128u : 0u;
            if constexpr (STATS) {
                const uint32_t fp = merge_flags(f0, f1, f2, f3) & vm;
                const unsigned c = __reduce_add_sync(
                    0xffffffffu, (unsigned)(__popc(fp & 0xC0C0C0C0u) | (__popc(fp & 0x30303030u) << 16)));
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
    extern __shared__ __align__(16) uint8_t smem[];
    // dynamic shared memory carve-up
    T* s_q = reinterpret_cast<T*>(smem);                                          // kTileQueries
    uint32_t* s_qsig = reinterpret_cast<uint32_t*>(s_q + kTileQueries);           // kTileQueries
    uint32_t* s_wsurv = s_qsig + kTileQueries;                                    // warps x kTileQueries (STATS)
    uint32_t* s_queue = s_wsurv + (STATS ? kScanWarps * kTileQueries : 0);        // warps x cap x 32
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t a_queue = smem_u32(s_queue) + 4u * (uint32_t)(warp * kLaneCap * 32 + lane);
    const uint32_t a_q = smem_u32(s_q), a_qsig = smem_u32(s_qsig);
    const uint32_t a_wsurv = smem_u32(s_wsurv + (STATS ? warp * kTileQueries : 0));
    unsigned long long surv_warp = 0;  // lane 0's copy is the warp total (STATS)
    OutChunk oc;

    for (uint32_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const Tile tl = tiles[t];
        __syncthreads();  // previous tile's shared state fully consumed
        for (uint32_t i = tid; i < tl.q_count; i += kScanThreads) {
            s_q[i] = (T)P.q_fp[tl.q_begin + i];
            s_qsig[i] = P.sig_on ? P.q_sig[tl.q_begin + i] : 0u;
        }
        T wc[kWordsPerLane];
        uint32_t wg[kWordsPerLane];
        uint32_t vmask = 0;
#pragma unroll
        for (int r = 0; r < kWordsPerLane; ++r) {
            const uint32_t widx = r * kScanThreads + tid;
            const bool ok = widx < tl.w_count;
            wc[r] = ok ? (T)P.w_fp[tl.w_begin + widx] : (T)0;
            wg[r] = ok && P.sig_on ? P.w_sig[tl.w_begin + widx] : 0u;
            // flag bits of word r = 4h + t for both queries: bit 8t + 7 - k, k = 2 qi + h
            if (ok) vmask |= (1u << (8 * (r & 3) + 7 - (r >> 2))) | (1u << (8 * (r & 3) + 5 - (r >> 2)));
        }
        __syncthreads();

        if (!tl.count_only) {
            TileScan<KIND, T, STATS> ts{P, tl, P.q_bytes + tl.q_bytes, P.w_bytes + tl.w_bytes,
                                        tl.q_len, tl.w_len, tl.q_stride, tl.w_stride,
                                        (tl.q_len <= 16 && tl.w_len <= 16) ? 1 : (tl.q_len <= 32 && tl.w_len <= 32) ? 2 : 0,
                                        tid, lane, a_queue, a_queue + 128u * (kLaneCap - 1), a_qsig, a_queue, oc};
            surv_warp += ts.scan(a_q, wc, wg, vmask, a_wsurv);
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
                    c += ((distance_of<KIND, T>(qc ^ wc[r], mf, ms, P.fold) <= P.thr) &&
                          (r * kScanThreads + tid < (int)tl.w_count)) ? 1u : 0u;
                c = __reduce_add_sync(0xffffffffu, c);
                if (lane == 0) s_wsurv[warp * kTileQueries + j] = c;
                surv_warp += c;
            }
        }
        if constexpr (STATS) {
            __syncthreads();
            for (uint32_t i = tid; i < tl.q_count; i += kScanThreads) {
                uint32_t v = 0;
#pragma unroll
                for (int w = 0; w < kScanWarps; ++w) v += s_wsurv[w * kTileQueries + i];
                if (v) atomicAdd(&P.q_survivors[P.q_ids[tl.q_begin + i]], v);
            }
        }
    }
    // run total of fingerprint survivors (reported), one atomic per warp
    if (STATS && lane == 0 && surv_warp) atomicAdd(P.survivors_total, surv_warp);
    oc.close(P.out, P.out_cap);
    if (lane == 0 && oc.real) atomicAdd(P.match_total, (unsigned long long)oc.real);
}

// Dynamic shared memory of k_scan<.., W, STATS>.
__host__ __device__ constexpr size_t scan_smem_bytes(int W, bool stats) {
    return (size_t)kTileQueries * (W <= 32 ? 4 : 8) + 4u * kTileQueries +
           (stats ? 4u * kScanWarps * kTileQueries : 0) + 4u * kScanWarps * kLaneCap * 32;
}

}  // namespace fpg
