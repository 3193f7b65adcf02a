// fpg_slice.cuh -- K2 as a bit-sliced scan (sm_100a): no POPC on the pair path.
//
// Layout.  The words of one dictionary length bucket, sorted by their eight
// group weights (input order within equal keys), are cut into slabs of 32
// consecutive words.  A slab is stored as NPT 32-bit planes:
// plane b holds bit b of the 32 words' comparison codes (K1b k_planes).
// Planes 0..NP-1 are the scheme fingerprint bits in the reference layout
// (fingerprint.hpp:48-56, :138-147: NF fields of FW bits above EXTRA one-bit
// fields); planes NP..NPT-1 are the "complement signature" sig' (below).
// In HBM a bucket's slabs are grouped into rows of 32 consecutive slabs, the
// unit a warp loads (lane = slab), and a row is plane-major: plane b of slab
// s at plane_base + (s / 32) * NPT * 32 + b * 32 + s % 32.  A lane reads its
// slab's NPT planes at compile-time offsets from one address, and every load
// of the warp is one coalesced 128-byte line.
//
// Test.  The reference rejects a pair iff ceil(F_D / 2) > k, i.e. F_D > 2k
// (dictionary.hpp:102-106, fingerprint.hpp:199,293-301), F_D = number of
// fields whose bits differ (ComparisonTables, fingerprint.hpp:171-214).  Here
// one lane evaluates it for the 32 words of a slab at once:
//   x_b   = plane_b XOR query_bit_b         one IMAD: plane * s + m with
//                                           (s, m) = (1, 0) or (-1, ~0), FMA pipe
//   x_f   = OR of the field's x_b           (LOP3, fields wider than 1 bit)
//   carry-save counter F = o + 2 t + 4 [f], fields entering four at a time:
//     o1 = o ^ x1 ^ x2, k1 = maj(o, x1, x2); o = o1 ^ x3 ^ x4,
//     k2 = maj(o1, x3, x4); f |= maj(t, k1, k2); t ^= k1 ^ k2   (7 LOP3)
// so bit w of f | (t & o) (k = 1: F >= 3; f | t | o for k = 0) says word w
// is rejected.  Per 32 pairs that is 7/4 ALU ops per 1-bit field plus the
// field ORs, and one IMAD per plane: about 1.6 ALU ops per comparison for
// count-16 with 16 sig' fields, against the POPC pipe's 16/clk/SM bound of a
// per-pair XOR + POPC.
//
// Scheduling.  A tile is (<= 128 queries) x (<= 256 slab groups of SL rows of
// 32 slabs) of one word length.  The tile's query masks are written to shared
// memory once; the warps then claim slab groups from a shared counter, load
// the group's planes into registers, build the group's query list through the
// weight window and scan it two queries per step.  Full-size tiles run
// between two CTA barriers (warp w's first group loads during the set-up);
// small batches take the instantiation without barriers (NB, below).
//
// Weight window.  sum_g |gw_g(q) - gw_g(x)| <= F_D over 8 field groups
// (fp_gweight), so a warp skips the queries whose group weights are more than
// 2k (L1) away from its slab group's weight box (k_group_box): those pairs
// are rejected by the reference test anyway.
//
// sig' (internal, exact).  Bytes that are NOT scheme letters are dealt into S
// extra one-bit occurrence fields (host LUT, frequency round robin).  One edit
// involves at most two symbols and each symbol owns at most one field of
// (scheme fields + sig' fields), so F_D + F_sig' <= 2 * distance for every
// variant / metric pair the reference filters with (occurrence, count:
// Hamming + Levenshtein; halved, position: Hamming).  Counting on through the
// sig' planes with the same counters therefore never drops a match; it only
// shrinks the candidate set the byte verifier sees.  QueryStats use the
// counters as they stand after the scheme planes (the reference's F_D alone)
// in the W = 32 / 64 kernels; W = 16 dictionaries take them from fingerprint
// histograms instead (k_fp_stats, fpg_kernels.cuh), and their kernels carry
// no survivor counters.
//
// Candidates (rare) go to a lane-private queue in shared memory as
// (query, slab row, 32-bit word mask) and leave the kernel as records of the
// candidate buffer; K3 (k_verify, fpg_verify.cuh) byte-verifies them at
// k <= 1 (edit_distance.hpp:18-64) right behind K2 and emits the matches as
// (query id << 32 | sorted word position) keys for K4, which maps positions
// to input-order ids.
#pragma once

#include <cstdint>
#include <type_traits>

namespace fpg {

// Device-side bounds checks for debug builds (FPG_DEBUG=1 python build.py).
#ifdef FPG_DEBUG
#define FPG_CHECK(c)                                                                           \
    do {                                                                                       \
        if (!(c)) {                                                                            \
            printf("FPG_CHECK failed %s:%d: %s (block %d thread %d)\n", __FILE__, __LINE__, #c, \
                   (int)blockIdx.x, (int)threadIdx.x);                                         \
            __trap();                                                                          \
        }                                                                                      \
    } while (0)
#else
#define FPG_CHECK(c) do { } while (0)
#endif

constexpr int kSliceThreads = 256;
constexpr int kSliceWarps = kSliceThreads / 32;
constexpr int kSliceQ = 128;      // queries per tile (shared-memory masks)
constexpr int kSliceCap = 8;      // queue entries per lane

__host__ __device__ constexpr int slice_slabs_per_lane(int npt) { return npt <= 40 ? 2 : 1; }
// Slabs per slab group: the unit a warp claims inside a tile (32 per lane row).
__host__ __device__ constexpr int slice_group_slabs(int npt) { return 32 * slice_slabs_per_lane(npt); }

struct SliceTile {
    uint32_t slab_begin;   // first slab of the tile, bucket-local
    uint32_t n_slabs;      // slabs in the tile (a multiple of the slab group but for a bucket's last tile)
    uint32_t q_begin;      // sorted query positions [q_begin, q_begin + q_count)
    uint32_t q_count;
    uint64_t plane_base;   // u32 offset of the bucket's planes
    uint64_t w_bytes;      // byte offset of the bucket in the padded word blob
    uint32_t ns;           // slabs in the bucket (plane row length)
    uint32_t w_start;      // sorted position of the bucket's first word
    uint32_t w_count;      // words in the bucket
    uint16_t w_len, w_stride;
    uint32_t count_only;   // fingerprint survivors counted, never verified
    uint32_t slab_g0;      // global index of the bucket's first slab (slab_w)
    uint32_t gbox_base;    // index in gbox of the tile's first slab group
    uint32_t pad_;
};

struct SliceParams {
    const uint32_t* planes;     // dictionary planes
    const uint64_t* q_fp;       // query fingerprints (sorted order)
    const uint32_t* q_sigp;     // query sig' codes
    const uint32_t* q_ids;
    const uint16_t* q_len;      // query lengths (sorted order)
    const uint32_t* q_start;    // per length: first sorted position
    const uint64_t* q_bbase;    // per length: byte offset in the padded query blob
    uint32_t* q_survivors;
    unsigned long long* survivors_total;
    unsigned int* tile_counter;
    int32_t k;
    int32_t stats;
    int32_t use_fp;             // scheme fields bound this metric (variant_supports, fingerprint.hpp:36-38)
    int32_t wskip;              // skip query / slab-group pairs whose weights differ by more than 2k
    const uint32_t* q_weight;   // per sorted query: group weights (fp_gweight, one nibble per group)
    const uint2* slab_w;        // per global slab: per-nibble min / max of its words' group weights
    const uint2* gbox;          // per slab group of a bucket (32 * SL slabs): the union of its slabs' boxes
    unsigned long long* scanned;  // pairs actually evaluated (after the weight skip)
    int32_t exhaustive;         // verify every pair: no fingerprint / sig' pruning (naive-path timing)
    int32_t drop_candidates;    // A/B diagnosis only (FPG_DROP_CANDIDATES=1): queued candidates are discarded unverified
    // candidate records for K3 (fpg_verify.cuh): cand_count = records reserved
    // (past cand_cap they are dropped and the host reruns)
    uint4* cand;
    unsigned long long* cand_count;
    uint64_t cand_cap;
    // the launch scans tiles tile_off + i * tile_stride, i < ntiles (round r of
    // R takes every R-th tile, so every round sees the plan's mix of lengths)
    uint32_t tile_off, tile_stride;
    int32_t no_barrier;         // tiles without CTA barriers (kernels whose double-buffered query data fits)
};

__device__ __forceinline__ int stride_of_len(int len) { return len <= 16 ? 16 : (len + 15) & ~15; }

// x = p XOR (query bit): s = 1, m = 0 keeps p; s = -1, m = ~0 gives ~p.
__device__ __forceinline__ uint32_t qxor(uint32_t p, uint32_t s, uint32_t m) { return p * s + m; }
// bitwise majority (the carry of a full adder): one LOP3
__device__ __forceinline__ uint32_t maj3(uint32_t a, uint32_t b, uint32_t c) { return (a & b) | (c & (a | b)); }
// One LOP3 with an explicit truth table (a = 0xf0, b = 0xcc, c = 0xaa).
template <uint32_t LUT>
__device__ __forceinline__ uint32_t lop3(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t d;
    asm("lop3.b32 %0, %1, %2, %3, %4;" : "=r"(d) : "r"(a), "r"(b), "r"(c), "n"(LUT));
    return d;
}
// Group weights are 8 nibbles (fp_gweight); the video intrinsics work on
// bytes, so even and odd nibbles are handled as two byte vectors.
constexpr uint32_t kNib = 0x0f0f0f0fu;
__device__ __forceinline__ uint32_t nib_min(uint32_t a, uint32_t b) {
    return __vminu4(a & kNib, b & kNib) | (__vminu4((a >> 4) & kNib, (b >> 4) & kNib) << 4);
}
__device__ __forceinline__ uint32_t nib_max(uint32_t a, uint32_t b) {
    return __vmaxu4(a & kNib, b & kNib) | (__vmaxu4((a >> 4) & kNib, (b >> 4) & kNib) << 4);
}
// Per-nibble min of lo and max of hi over the warp: a group-weight box.
__device__ __forceinline__ uint2 warp_box(uint32_t lo, uint32_t hi) {
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
        lo = nib_min(lo, __shfl_xor_sync(0xffffffffu, lo, d));
        hi = nib_max(hi, __shfl_xor_sync(0xffffffffu, hi, d));
    }
    return make_uint2(lo, hi);
}
// A box split into even / odd nibble byte vectors: (lo even, lo odd, hi even, hi odd).
__device__ __forceinline__ uint4 split_box(uint2 box) {
    return make_uint4(box.x & kNib, (box.x >> 4) & kNib, box.y & kNib, (box.y >> 4) & kNib);
}
// L1 distance between a query's group weights (split: even, odd nibbles) and
// a split box: at most one of the two saturated differences of a group is
// non-zero.
__device__ __forceinline__ uint32_t box_dist(uint32_t qe, uint32_t qo, uint4 b) {
    return __vsadu4(__vsubus4(b.x, qe) | __vsubus4(qe, b.z), 0u) + __vsadu4(__vsubus4(b.y, qo) | __vsubus4(qo, b.w), 0u);
}

template <int NP, int FW, int EXTRA, int S>
struct SliceShape {
    static constexpr int NPT = NP + S;
    static constexpr int SL = slice_slabs_per_lane(NPT);
    static constexpr int NF = (NP - EXTRA) / FW;
    static_assert(NF * FW + EXTRA == NP, "field layout");
    static_assert(NPT % 2 == 0, "plane pairs");
};

// Tiles without CTA barriers (below): the tile's query data is double
// buffered, which fits two CTAs per SM while the masks are small enough.
__host__ __device__ constexpr bool slice_no_barrier(int npt) { return npt <= 40; }
// Dynamic shared memory of k_slice<NP, .., S>.
__host__ __device__ constexpr size_t slice_smem_bytes(int npt, bool nb) {
    return ((size_t)kSliceQ * npt * 8 + 12u * kSliceQ) * (nb ? 2 : 1) + 8u * kSliceCap * kSliceThreads +
           2u * kSliceQ * kSliceWarps;
}
// Flags between the warps of a CTA (shared memory, CTA scope).
__device__ __forceinline__ uint32_t ld_acquire_cta(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.cta.shared.u32 %0, [%1];" : "=r"(v) : "r"((uint32_t)__cvta_generic_to_shared(p)) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_cta(uint32_t* p, uint32_t v) {
    asm volatile("st.release.cta.shared.u32 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(p)), "r"(v) : "memory");
}

// HOT: the options of the common run fixed at compile time (fingerprint
// filter on, weight window on, k = 1, not exhaustive; survivor counters for
// QueryStats on for W = 32 / 64 and off for W = 16, whose stats come from the
// fingerprint histograms, k_fp_stats), so the per-step code carries no
// uniform branches on them; other runs take the generic instantiation
// (HOT = false), which reads them from P.
//
// X (position-code path, Hamming; instantiated with NP = 0): the planes are
// the symbol codes of kXLen byte positions of each word, kXBits planes per
// position (every position of a word of <= kXLen bytes, else positions spread
// over the word, k_build), and q_sigp holds the queries' codes.  The counters
// count the positions whose codes differ, and a word is a candidate iff at
// most k of them differ: exactly hamming_bounded's test
// (edit_distance.hpp:18-27) for words of <= kXLen bytes, a sound filter for
// longer ones (K3 decides).  No scheme planes, no survivor counters: the host
// takes the path only when QueryStats come from the histograms.
template <int NP, int FW, int EXTRA, int S, bool HOT, bool X = false, bool NB = false>
__global__ void __launch_bounds__(kSliceThreads, 2) k_slice(const SliceTile* __restrict__ tiles, uint32_t ntiles,
                                                            const __grid_constant__ SliceParams P) {
    using Sh = SliceShape<NP, FW, EXTRA, S>;
    constexpr int NPT = Sh::NPT, SL = Sh::SL, NF = Sh::NF;
    const bool o_use_fp = HOT || P.use_fp;
    // HOT kernels of W = 16 dictionaries carry no survivor counters: the host
    // takes QueryStats::verified from the fingerprint histograms (k_fp_stats)
    // (the exact path's kernel has no scheme planes: never any counters)
    const bool o_stats = X ? false : HOT ? (NP > 16) : (P.stats != 0);
    const bool o_wskip = HOT || P.wskip;
    const bool o_exhaustive = !HOT && P.exhaustive;
    const int o_k = HOT ? 1 : P.k;
    // NB: no CTA barrier per tile.  The tile's query data (masks, ids, byte
    // offsets, lengths, weights, survivor counts, group counter) lives in two
    // buffers used by alternate tiles.  The first warp to run out of groups in
    // tile n claims the set-up of tile n + 1 (a CAS on s_claim), waits until
    // every warp has left tile n - 1 (the buffer's previous user; its last
    // leaver also posts the tile's per-query survivor counts), fills the
    // buffer alone and publishes it; the other warps move on to tile n + 1
    // as they finish, so nobody waits for the tile's slowest slab group.
    // The host picks it per launch (P.no_barrier): small batches, whose tiles
    // hold a few slab groups per warp, lose up to 15% of K2 to the barrier;
    // full-size tiles (config 5) run 0-4% faster with it, since the barrier
    // variant loads each warp's first group during the set-up.
    // Two instantiations: the launcher takes NB when P.no_barrier is set and
    // the double buffers fit (a run-time switch inside one kernel cost the
    // full-size tiles 3-7%).
    static_assert(!NB || slice_no_barrier(NPT), "double-buffered query data must fit");
    constexpr int NBUF = NB ? 2 : 1;
    constexpr uint32_t kEndTile = 0xffffffffu;
    extern __shared__ __align__(16) uint8_t smem[];
    uint2* s_qm_all = reinterpret_cast<uint2*>(smem);                                     // [NBUF][kSliceQ][NPT] (s, m)
    uint32_t* s_qid_all = reinterpret_cast<uint32_t*>(s_qm_all + NBUF * kSliceQ * NPT);   // [NBUF][kSliceQ]: input query id
    uint32_t* s_qoff_all = s_qid_all + NBUF * kSliceQ;                                    // [NBUF][kSliceQ]: byte offset / 16 in the query blob
    uint32_t* s_qlen_all = s_qoff_all + NBUF * kSliceQ;                                   // [NBUF][kSliceQ]: length
    uint2* s_queue = reinterpret_cast<uint2*>(s_qlen_all + NBUF * kSliceQ);               // [cap][threads]
    uint16_t* s_qlist = reinterpret_cast<uint16_t*>(s_queue + kSliceCap * kSliceThreads);  // [warps][kSliceQ]
    __shared__ uint32_t s_grp_all[NBUF];  // next slab group of the tile
    __shared__ uint32_t s_next[2];  // next tile index, double-buffered by iteration parity (barrier variant)
    __shared__ uint32_t s_surv_all[NBUF][kSliceQ];
    __shared__ uint32_t s_qw_all[NBUF][2][kSliceQ];  // query group weights: even, odd nibbles (byte vectors)
    // NB flags, per buffer: the tile it holds, completed set-ups, retired
    // uses, warps that have left the current use; s_claim: next tile
    // iteration whose set-up nobody has claimed
    __shared__ uint32_t s_tile[2], s_ready[2], s_retired[2], s_done[2], s_claim;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    unsigned long long surv_warp = 0;  // lanes 0, 1: the warp's fingerprint survivors
    unsigned long long scanned_warp = 0;  // lane 0

    // query (s, m) masks, ids, byte offsets and group weights of a tile into
    // buffer p; query j0, j0 + jstep, ... by the calling thread
    auto setup = [&](int p, const SliceTile& tq, uint32_t j0, uint32_t jstep) {
        uint2* qm_p = s_qm_all + p * kSliceQ * NPT;
        for (uint32_t j = j0; j < tq.q_count; j += jstep) {
            const uint32_t qp = tq.q_begin + j;
            const uint64_t f = __ldg(P.q_fp + qp);
            const uint32_t g = __ldg(P.q_sigp + qp);
            const uint32_t id = P.q_ids[qp];
            uint2* dst = qm_p + j * NPT;
#pragma unroll
            for (int b = 0; b < NPT; ++b) {
                const uint32_t bit = b < NP ? (uint32_t)(f >> b) & 1u : (g >> (b - NP)) & 1u;
                dst[b] = bit ? make_uint2(0xffffffffu, 0xffffffffu) : make_uint2(1u, 0u);
            }
            s_qid_all[p * kSliceQ + j] = id;
            const int m = P.q_len[qp];
            s_qlen_all[p * kSliceQ + j] = (uint32_t)m;
            s_qoff_all[p * kSliceQ + j] = (uint32_t)((P.q_bbase[m] + (uint64_t)(qp - P.q_start[m]) * stride_of_len(m)) >> 4);
            s_surv_all[p][j] = 0u;
            const uint32_t qw = o_wskip ? P.q_weight[qp] : 0u;
            s_qw_all[p][0][j] = qw & kNib;
            s_qw_all[p][1][j] = (qw >> 4) & kNib;
        }
    };
    // NB: one warp claims the next tile and sets up iteration n in buffer n & 1
    auto setup_next = [&](uint32_t n) {
        const int p = (int)(n & 1u);
        if (lane == 0)
            while (ld_acquire_cta(&s_retired[p]) != (n >> 1)) __nanosleep(32);
        __syncwarp();
        uint32_t tn = 0;
        if (lane == 0) tn = atomicAdd(P.tile_counter, 1u);
        tn = __shfl_sync(0xffffffffu, tn, 0);
        if (tn < ntiles) {
            const SliceTile tq = tiles[(uint64_t)tn * P.tile_stride + P.tile_off];
            setup(p, tq, (uint32_t)lane, 32u);
        }
        if (lane == 0) {
            s_tile[p] = tn < ntiles ? tn : kEndTile;
            s_grp_all[p] = 0u;
        }
        __threadfence_block();
        __syncwarp();
        if (lane == 0) st_release_cta(&s_ready[p], (n >> 1) + 1u);
    };

    uint32_t t = 0;
    if constexpr (NB) {
        if (tid == 0) {
            s_ready[0] = s_ready[1] = s_retired[0] = s_retired[1] = s_done[0] = s_done[1] = 0u;
            s_claim = 1u;  // iteration 0 is set up by warp 0 right here
        }
        __syncthreads();
        if (warp == 0) setup_next(0u);
    } else {
        if (tid == 0) s_next[0] = atomicAdd(P.tile_counter, 1u);
        __syncthreads();
        t = s_next[0];
    }
    for (uint32_t it = NB ? 0u : 1u;; ++it) {
        const int pb = NB ? (int)(it & 1u) : 0;  // this tile's buffer
        if constexpr (NB) {
            if (lane == 0)
                while (ld_acquire_cta(&s_ready[pb]) != (it >> 1) + 1u) __nanosleep(32);
            __syncwarp();
            t = s_tile[pb];
            if (t == kEndTile) break;
        } else {
            if (t >= ntiles) break;
        }
        const SliceTile tl = tiles[(uint64_t)t * P.tile_stride + P.tile_off];
        uint2* const s_qm = s_qm_all + pb * kSliceQ * NPT;
        uint32_t* const s_qid = s_qid_all + pb * kSliceQ;
        uint32_t* const s_qoff = s_qoff_all + pb * kSliceQ;
        uint32_t* const s_qlen = s_qlen_all + pb * kSliceQ;
        uint32_t* const s_surv = s_surv_all[pb];
        uint32_t(*const s_qw)[kSliceQ] = s_qw_all[pb];
        uint32_t* const s_grp = &s_grp_all[pb];
        if constexpr (!NB) {
            if (tid == 0) s_next[it & 1] = atomicAdd(P.tile_counter, 1u);  // read after the end-of-tile barrier
            setup(0, tl, (uint32_t)tid, (uint32_t)kSliceThreads);  // one query per thread
        }
        // this lane's slabs of slab group g (SL rows of 32 slabs), the
        // group's valid words and its group-weight box
        uint32_t pl[SL][NPT];
        uint32_t valid[SL];
        const uint32_t* planes = P.planes + tl.plane_base;  // the tile's bucket
        uint32_t vw = 0;
        uint2 box = make_uint2(0u, 0u);
        const uint32_t n_grp = (tl.n_slabs + 32u * SL - 1u) / (32u * SL);
        auto load_group = [&](uint32_t g) {
            uint32_t wlo = 0xffffffffu, whi = 0u;
            vw = 0;
#pragma unroll
            for (int r = 0; r < SL; ++r) {
                const uint32_t rel = 32u * (SL * g + r) + (uint32_t)lane;
                const uint32_t slab = tl.slab_begin + rel;
                const bool ok = rel < tl.n_slabs;
                // lanes past the tile's end load the tile's first slab (valid
                // memory; valid[r] = 0 masks every result of theirs).  Rows of
                // 32 slabs are plane-major: one address per row, the planes at
                // compile-time offsets
                const uint32_t sl_ = ok ? slab : tl.slab_begin;
                const uint32_t* src = planes + (uint64_t)(sl_ >> 5) * (NPT * 32) + (sl_ & 31u);
#pragma unroll
                for (int b = 0; b < NPT; ++b) pl[r][b] = __ldg(src + 32 * b);
                const uint32_t rem = tl.w_count - 32u * slab;  // words left in the bucket from this slab on
                valid[r] = !ok ? 0u : rem >= 32u ? 0xffffffffu : ((1u << rem) - 1u);
                vw += __popc(valid[r]);
            }
            // the group's weight box, precomputed at construction (k_group_box)
            box = o_wskip ? __ldg(P.gbox + tl.gbox_base + g) : make_uint2(wlo, whi);
        };
        // barrier variant: warp w's first group is group w, its planes load
        // while the queries are set up; later groups (NB: all groups) are
        // claimed from s_grp
        uint32_t g = (uint32_t)warp;
        if constexpr (!NB) {
            if (g < n_grp) load_group(g);
            if (tid == 0) *s_grp = (uint32_t)kSliceWarps;
            __syncthreads();
        }

        // The lane's queue is addressed by a running shared-memory pointer
        // (32-bit window address): a push is one store and one add.
        const uint32_t qbase = (uint32_t)__cvta_generic_to_shared(s_queue + tid);
        constexpr uint32_t kQStep = 8u * kSliceThreads;  // bytes between a lane's slots
        uint32_t qtop = qbase;  // next free slot
        const bool verify = !tl.count_only;

        // Hands the warp's queued (query, slab row, mask) entries to K3
        // (fpg_verify.cuh): the lanes' entries become self-describing records
        // in the candidate buffer, reserved with one atomic per flush.  A
        // reservation past the buffer's end is dropped: the count tells the
        // host, which reruns the batch with a larger buffer or in more rounds.
        auto flush = [&]() {
            __syncwarp();
            const uint32_t qn = (qtop - qbase) / kQStep;  // queued entries of this lane
            qtop = qbase;
            if (P.drop_candidates) return;
            uint32_t incl = qn;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const uint32_t v = __shfl_up_sync(0xffffffffu, incl, d);
                if (lane >= d) incl += v;
            }
            const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
            if (total == 0) return;
            unsigned long long base = 0;
            if (lane == 31) base = atomicAdd(P.cand_count, (unsigned long long)total);
            base = __shfl_sync(0xffffffffu, base, 31);
            if (base + total <= P.cand_cap) {
                uint4* dst = P.cand + base + (incl - qn);
                // byte offset / 16 of word 0 of this lane's slab in tile slab row 0,
                // and of one slab row (1024 words)
                const uint32_t s16 = (uint32_t)tl.w_stride >> 4;
                const uint32_t w0 = (uint32_t)(tl.w_bytes >> 4) + 32u * (tl.slab_begin + (uint32_t)lane) * s16;
#pragma unroll 1
                for (uint32_t s = 0; s < qn; ++s) {
                    const uint2 e = s_queue[s * kSliceThreads + tid];
                    const uint32_t j = e.x & 0xffffu;
                    FPG_CHECK(j < tl.q_count && 32u * (e.x >> 16) < tl.n_slabs);
                    dst[s] = make_uint4(s_qoff[j], w0 + 1024u * s16 * (e.x >> 16), e.y, (uint32_t)tl.w_len | (s_qlen[j] << 16));
                }
            }
        };

        // Per-warp slab count: warps whose second slab row is empty (a
        // bucket's last chunk) run the one-slab loop instead of scanning zeros.
        // One step = NQ consecutive queries (j .. j + NQ - 1) against the
        // lane's SLX slabs: NQ * SLX independent counter chains per plane.
        // step over list entries i .. i + NQ - 1 (tile query indices)
        const uint16_t* qlist = s_qlist + warp * kSliceQ;
        uint32_t row0 = 0;  // tile slab row of this lane's pl[0]
        auto step = [&](auto slc, auto nqc, uint32_t i) {
            constexpr int SLX = decltype(slc)::value;
            constexpr int NQ = decltype(nqc)::value;
            const uint4* qm[NQ];
            uint32_t jq[NQ];
#pragma unroll
            for (int h = 0; h < NQ; ++h) {
                jq[h] = qlist[i + h];
                qm[h] = reinterpret_cast<const uint4*>(s_qm + jq[h] * NPT);
            }
            // Carry-save saturating counter per word: F = o + 2 t + 4 [f], i.e.
            // o = ones bit, t = twos bit, f = "F >= 4".  Field bits enter four
            // at a time (two full adders into o, one into t: 7 LOP3 per 4
            // fields) or two at a time (4 LOP3); reject at k = 1 is
            // F >= 3 = f | (t & o), at k = 0 F >= 1 = f | t | o.  f starts as
            // the complement of the valid words (a slab's words past the
            // bucket's end are rejected), so a pass / candidate mask is one
            // LOP3: ~(f | (t & o)).
            uint32_t co[NQ][SLX], ct[NQ][SLX], cf[NQ][SLX];
#pragma unroll
            for (int h = 0; h < NQ; ++h)
#pragma unroll
                for (int r = 0; r < SLX; ++r) {
                    co[h][r] = ct[h][r] = 0u;
                    cf[h][r] = ~valid[r];  // folded into the first LOP3 that reads it
                }
            // (s, m) of plane b for query h
#define FPG_QS(h, b) ((b) & 1 ? qm[h][(b) >> 1].z : qm[h][(b) >> 1].x)
#define FPG_QM(h, b) ((b) & 1 ? qm[h][(b) >> 1].w : qm[h][(b) >> 1].y)
            // field i of the code as a 32-word "differs" mask: scheme fields
            // (NF fields of FW planes, then EXTRA one-bit fields), then sig'
            auto fbit = [&](int h, int r, int i) -> uint32_t {
                if (i < NF) {
                    const int b0 = EXTRA + FW * i;
                    uint32_t x = qxor(pl[r][b0], FPG_QS(h, b0), FPG_QM(h, b0));
                    if constexpr (FW % 2 == 0) {
                        // even widths: the last plane joins the OR as x | (p ^ m),
                        // one LOP3 either way, so its query XOR needs no IMAD
#pragma unroll
                        for (int u = 1; u + 1 < FW; ++u) x |= qxor(pl[r][b0 + u], FPG_QS(h, b0 + u), FPG_QM(h, b0 + u));
                        x |= pl[r][b0 + FW - 1] ^ FPG_QM(h, b0 + FW - 1);
                    } else {
#pragma unroll
                        for (int u = 1; u < FW; ++u) x |= qxor(pl[r][b0 + u], FPG_QS(h, b0 + u), FPG_QM(h, b0 + u));
                    }
                    return x;
                }
                if constexpr (X) {
                    if (i >= NF + EXTRA) {  // byte position p: its kXBits code planes differ anywhere
                        const int b0 = NP + kXBits * (i - NF - EXTRA);
                        uint32_t x = qxor(pl[r][b0], FPG_QS(h, b0), FPG_QM(h, b0));
#pragma unroll
                        for (int u = 1; u < kXBits; ++u) x |= qxor(pl[r][b0 + u], FPG_QS(h, b0 + u), FPG_QM(h, b0 + u));
                        return x;
                    }
                }
                const int b = i < NF + EXTRA ? i - NF : NP + (i - NF - EXTRA);
                return qxor(pl[r][b], FPG_QS(h, b), FPG_QM(h, b));
            };
            // mode 0: f |= m; 1: m is held back (pm); 2: f |= pm | m (one LOP3
            // for two quads' fours carries)
            uint32_t pm[NQ][SLX];
            auto add4 = [&](int h, int r, uint32_t x1, uint32_t x2, uint32_t x3, uint32_t x4, int mode) {
                const uint32_t o = co[h][r];
                const uint32_t o1 = o ^ x1 ^ x2, k1 = maj3(o, x1, x2);
                const uint32_t k2 = maj3(o1, x3, x4);
                co[h][r] = o1 ^ x3 ^ x4;
                const uint32_t t = ct[h][r];
                const uint32_t m = maj3(t, k1, k2);
                if (mode == 1) pm[h][r] = m;
                else if (mode == 2) cf[h][r] |= pm[h][r] | m;
                else cf[h][r] |= m;
                ct[h][r] = t ^ k1 ^ k2;
            };
            auto add2 = [&](int h, int r, uint32_t x1, uint32_t x2) {
                const uint32_t o = co[h][r], k1 = maj3(o, x1, x2);
                co[h][r] = o ^ x1 ^ x2;
                cf[h][r] |= ct[h][r] & k1;
                ct[h][r] ^= k1;
            };
            // fields [i0, i1) into the counters
            auto count = [&](auto i0c, auto i1c) {
                constexpr int I0 = decltype(i0c)::value, I1 = decltype(i1c)::value;
                constexpr int N4 = (I1 - I0) / 4 * 4;
#pragma unroll
                for (int i = I0; i < I0 + N4; i += 4) {
                    const int q = (i - I0) / 4;  // quad index: pairs of quads share the carry OR
                    const int mode = (q & 1) ? 2 : (q + 1 < N4 / 4 ? 1 : 0);
#pragma unroll
                    for (int h = 0; h < NQ; ++h)
#pragma unroll
                        for (int r = 0; r < SLX; ++r)
                            add4(h, r, fbit(h, r, i), fbit(h, r, i + 1), fbit(h, r, i + 2), fbit(h, r, i + 3), mode);
                }
#pragma unroll
                for (int i = I0 + N4; i < I1; i += 2)
#pragma unroll
                    for (int h = 0; h < NQ; ++h)
#pragma unroll
                        for (int r = 0; r < SLX; ++r) add2(h, r, fbit(h, r, i), i + 1 < I1 ? fbit(h, r, i + 1) : 0u);
            };
            // words that pass: ~(f | (t & o)) at k = 1, ~(f | t | o) at k = 0 (one LOP3)
            auto passed = [&](int h, int r) -> uint32_t {
                return o_k ? lop3<0x07>(cf[h][r], ct[h][r], co[h][r]) : lop3<0x01>(cf[h][r], ct[h][r], co[h][r]);
            };
            // scheme fields.  Skipped when they do not bound the metric (halved
            // / position with Levenshtein, filter off): sig' alone stays a
            // valid bound.
            // (the exact path counts them for QueryStats only)
            if (o_use_fp && (!X || o_stats)) count(std::integral_constant<int, 0>{}, std::integral_constant<int, NF + EXTRA>{});
            if (o_stats) {  // fingerprint survivors: QueryStats::verified (dictionary.hpp:102-110)
                uint32_t sv = 0;  // query h in bits [16 h, 16 h + 16): <= 2048 per warp
#pragma unroll
                for (int h = 0; h < NQ; ++h)
#pragma unroll
                    for (int r = 0; r < SLX; ++r) sv += (uint32_t)__popc(passed(h, r)) << (16 * h);
                sv = __reduce_add_sync(0xffffffffu, sv);
                static_assert(NQ <= 2, "two queries per step at most");
                if (lane < NQ) {
                    const uint32_t v = (sv >> (16 * lane)) & 0xffffu;
                    if (v) atomicAdd(&s_surv[lane ? jq[NQ - 1] : jq[0]], v);
                    surv_warp += v;
                }
            }
            if (verify) {
                if constexpr (X) {
                    static_assert(S == kXBits * kXLen, "exact path planes");
#pragma unroll
                    for (int h = 0; h < NQ; ++h)
#pragma unroll
                        for (int r = 0; r < SLX; ++r) {
                            co[h][r] = ct[h][r] = 0u;
                            cf[h][r] = ~valid[r];
                        }
                    count(std::integral_constant<int, NF + EXTRA>{}, std::integral_constant<int, NF + EXTRA + kXLen>{});
                } else if (!o_exhaustive) {
                    count(std::integral_constant<int, NF + EXTRA>{}, std::integral_constant<int, NF + EXTRA + S>{});
                }
                // exact path: at most k differing positions, ~(f | t) at k = 1
                auto exact_pass = [&](int h, int r) -> uint32_t {
                    return o_k ? lop3<0x03>(cf[h][r], ct[h][r], 0u) : lop3<0x01>(cf[h][r], ct[h][r], co[h][r]);
                };
#pragma unroll
                for (int h = 0; h < NQ; ++h)
#pragma unroll
                    for (int r = 0; r < SLX; ++r) {
                        const uint32_t cand = X ? exact_pass(h, r) : o_exhaustive ? valid[r] : passed(h, r);
                        if (cand) {
                            asm volatile("st.shared.v2.u32 [%0], {%1, %2};" ::"r"(qtop), "r"(jq[h] | ((row0 + (uint32_t)r) << 16)),
                                         "r"(cand)
                                         : "memory");
                            qtop += kQStep;
                        }
                    }
                // room for the largest step (2 queries x SL slabs) whatever comes next
                if (__any_sync(0xffffffffu, qtop > qbase + (uint32_t)(kSliceCap - 2 * SL) * kQStep)) flush();
            }
#undef FPG_QS
#undef FPG_QM
        };
        // Slab groups (SL rows of 32 slabs) are claimed one at a time from
        // s_grp: no barrier between them, so the warps of a tile stay busy
        // whatever the weight window leaves per group, and the tile's query
        // masks serve all of its groups.  Per group: the lane's slab planes
        // into registers, the group's weight box, and the list of tile queries
        // whose group weights are within L1 distance 2k of the box (the others
        // have F_D > 2k with every word of the group: sum_g |group weight
        // difference| <= F_D).
        {
            const uint32_t span = 2u * (uint32_t)o_k;
            uint16_t* ql = s_qlist + warp * kSliceQ;
            for (bool first = !NB;; first = false) {
                if (!first) {
                    if (lane == 0) g = atomicAdd(s_grp, 1u);
                    g = __shfl_sync(0xffffffffu, g, 0);
                    if (g < n_grp) load_group(g);
                }
                if (g >= n_grp) break;
                row0 = (uint32_t)SL * g;
                const uint4 sbox = split_box(box);
                uint32_t nlist = 0;
                for (uint32_t b = 0; b < tl.q_count; b += 32) {
                    const uint32_t j = b + (uint32_t)lane;
                    bool in = j < tl.q_count;
                    if (in && o_wskip) in = box_dist(s_qw[0][j], s_qw[1][j], sbox) <= span;
                    const uint32_t bal = __ballot_sync(0xffffffffu, in);
                    if (in) ql[nlist + __popc(bal & ((1u << lane) - 1u))] = (uint16_t)j;
                    nlist += __popc(bal);
                }
                __syncwarp();
                // pairs actually evaluated (stats / roofline)
                const uint32_t vws = __reduce_add_sync(0xffffffffu, vw);
                if (lane == 0 && verify) scanned_warp += (unsigned long long)vws * nlist;
                uint32_t i = 0;
                if (SL == 2 && 32u * (row0 + 1u) < tl.n_slabs) {
                    if constexpr (NPT <= 48)  // query pairs while the registers allow it
                        for (; i + 2 <= nlist; i += 2) step(std::integral_constant<int, SL>{}, std::integral_constant<int, 2>{}, i);
                    for (; i < nlist; ++i) step(std::integral_constant<int, SL>{}, std::integral_constant<int, 1>{}, i);
                } else {
                    if constexpr (NPT <= 48)
                        for (; i + 2 <= nlist; i += 2) step(std::integral_constant<int, 1>{}, std::integral_constant<int, 2>{}, i);
                    for (; i < nlist; ++i) step(std::integral_constant<int, 1>{}, std::integral_constant<int, 1>{}, i);
                }
            }
        }
        if (verify) flush();
        if constexpr (NB) {
            // leave the tile: the last warp out posts the survivor counts and
            // retires the buffer; the first one out sets up the next tile
            __threadfence_block();
            __syncwarp();
            uint32_t left = 0;
            if (lane == 0) left = atomicAdd(&s_done[pb], 1u);
            left = __shfl_sync(0xffffffffu, left, 0);
            if (left == (uint32_t)kSliceWarps - 1u) {
                __threadfence_block();
                if (o_stats)
                    for (uint32_t j = (uint32_t)lane; j < tl.q_count; j += 32u)
                        if (s_surv[j]) atomicAdd(&P.q_survivors[s_qid[j]], s_surv[j]);
                __syncwarp();
                if (lane == 0) {
                    s_done[pb] = 0u;
                    st_release_cta(&s_retired[pb], (it >> 1) + 1u);
                }
            }
            uint32_t won = 0;
            if (lane == 0) won = atomicCAS(&s_claim, it + 1u, it + 2u) == it + 1u;
            if (__shfl_sync(0xffffffffu, won, 0)) setup_next(it + 1u);
        } else {
            __syncthreads();  // tile consumed; s_next[it & 1] and s_surv complete
            if (o_stats)
                for (uint32_t j = tid; j < tl.q_count; j += kSliceThreads)
                    if (s_surv[j]) atomicAdd(&P.q_survivors[s_qid[j]], s_surv[j]);
            t = s_next[it & 1];
        }
    }
    if (o_stats && lane < 2 && surv_warp) atomicAdd(P.survivors_total, surv_warp);
    if (lane == 0 && scanned_warp) atomicAdd(P.scanned, scanned_warp);
}

// ---------------------------------------------------------------- K1b planes
// One warp per slab: lane i holds word 32 s + i of its bucket; plane b is the
// ballot of bit b of the words' codes (fingerprint bits, then sig' bits).  A
// CTA of kPlanesSlabs warps handles that many consecutive global slabs and
// stores each plane row through shared memory, so a row of consecutive slabs
// leaves as one coalesced store instead of one 4-byte word per warp.
constexpr int kPlanesSlabs = 32;  // warps (= consecutive slabs) per CTA
#ifndef FPG_K2_TU  // defined once, in fpg_api.cu
__global__ void __launch_bounds__(32 * kPlanesSlabs) k_planes(
    const uint64_t* __restrict__ fp, const uint32_t* __restrict__ sigp, const uint32_t* __restrict__ weight,
    uint2* __restrict__ slab_w,
    const uint32_t* __restrict__ slab_start,  // per length: first global slab (L1 + 1)
    const uint32_t* __restrict__ start,       // per length: first sorted position
    const uint32_t* __restrict__ count,       // per length: words
    const uint64_t* __restrict__ plane_base,  // per length: u32 offset of the planes
    int nlen, uint32_t total_slabs, int np, int npt, uint32_t* __restrict__ planes) {
    __shared__ uint32_t tile[96][kPlanesSlabs + 1];  // [plane][slab of the CTA]
    __shared__ int s_l0;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const uint32_t gs0 = blockIdx.x * kPlanesSlabs;
    const uint32_t gs = gs0 + (uint32_t)w;
    // bucket of the CTA's first slab (largest L with slab_start[L] <= gs0),
    // searched once; the CTA's 32 slabs reach at most a few buckets further
    if (threadIdx.x == 0) {
        int lo = 0, hi = nlen;
        while (hi - lo > 1) {
            const int mid = (lo + hi) >> 1;
            if (slab_start[mid] <= gs0) lo = mid;
            else hi = mid;
        }
        s_l0 = lo;
    }
    __syncthreads();
    auto bucket = [&](uint32_t g) {
        int L = s_l0;
        while (slab_start[L + 1] <= g) ++L;
        return L;
    };
    if (gs < total_slabs) {
        const int L = bucket(gs);
        const uint32_t s = gs - slab_start[L];
        const uint32_t wi = 32u * s + lane;
        const bool ok = wi < count[L];
        const uint64_t f = ok ? fp[start[L] + wi] : 0ull;
        const uint32_t g = ok ? sigp[start[L] + wi] : 0u;
        if (slab_w) {  // the slab's group-weight box (K2's weight window): per-nibble min / max
            const uint32_t wt = ok ? weight[start[L] + wi] : 0u;
            const uint2 box = warp_box(ok ? wt : 0xffffffffu, ok ? wt : 0u);
            if (lane == 0) slab_w[gs] = box;
        }
        for (int b = 0; b < npt; ++b) {  // warp-uniform
            const uint32_t bit = b < np ? (uint32_t)(f >> b) & 1u : (g >> (b - np)) & 1u;
            const uint32_t ball = __ballot_sync(0xffffffffu, bit != 0);
            if (lane == 0) tile[b][w] = ball;
        }
    }
    __syncthreads();
    // rows: element (b, slab gs0 + i), i = lane; consecutive lanes write
    // consecutive slabs of one bucket's plane row
    for (int b = w; b < npt; b += kPlanesSlabs) {
        const uint32_t g = gs0 + (uint32_t)lane;
        if (g < total_slabs) {
            const int L = bucket(g);
            const uint32_t sl = g - slab_start[L];  // row of 32 slabs, plane-major inside
            planes[plane_base[L] + (uint64_t)(sl >> 5) * ((uint32_t)npt * 32u) + (uint32_t)b * 32u + (sl & 31u)] = tile[b][lane];
        }
    }
}
#endif

// Weight box of every slab group (gsl consecutive slabs of a bucket, the unit
// a K2 warp claims): per-nibble min / max over its slabs' boxes.  One thread
// per group.
#ifndef FPG_K2_TU  // defined once, in fpg_api.cu
__global__ void k_group_box(const uint2* __restrict__ slab_w, const uint32_t* __restrict__ slab_start,
                            const uint32_t* __restrict__ group_start, int nlen, uint32_t total_groups, uint32_t gsl,
                            uint2* __restrict__ gbox) {
    const uint32_t gi = blockIdx.x * blockDim.x + threadIdx.x;
    if (gi >= total_groups) return;
    int lo = 0, hi = nlen;  // bucket: largest L with group_start[L] <= gi
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (group_start[mid] <= gi) lo = mid;
        else hi = mid;
    }
    const uint32_t ns = slab_start[lo + 1] - slab_start[lo];
    const uint32_t s0 = (gi - group_start[lo]) * gsl;
    uint32_t wlo = 0xffffffffu, whi = 0u;
    for (uint32_t s = s0; s < s0 + gsl && s < ns; ++s) {
        const uint2 mm = slab_w[slab_start[lo] + s];
        wlo = nib_min(wlo, mm.x);
        whi = nib_max(whi, mm.y);
    }
    gbox[gi] = make_uint2(wlo, whi);
}
#endif

// 256-bin byte histogram of a blob (sig' symbol ranking).
#ifndef FPG_K2_TU  // defined once, in fpg_api.cu
__global__ void k_hist256(const uint8_t* __restrict__ blob, uint64_t n, unsigned long long* __restrict__ hist) {
    __shared__ unsigned int h[256];
    h[threadIdx.x] = 0;  // blockDim == 256
    __syncthreads();
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        atomicAdd(&h[blob[i]], 1u);
    __syncthreads();
    if (h[threadIdx.x]) atomicAdd(&hist[threadIdx.x], (unsigned long long)h[threadIdx.x]);
}
#endif

}  // namespace fpg
