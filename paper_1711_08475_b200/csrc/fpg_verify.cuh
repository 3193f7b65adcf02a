// fpg_verify.cuh -- K3: out-of-line byte verification of K2's candidates
// (sm_100a).
//
// The bit-sliced K2 (fpg_slice.cuh) does not verify its candidates itself.
// Every (query, slab, 32-word mask) entry that survives the fingerprint and
// sig' (or exact) planes leaves K2 as one self-describing 16-byte record in
// the candidate buffer:
//     x = byte offset / 16 of the query in the padded query blob
//     y = byte offset / 16 of the slab's word 0 in the padded word blob
//     z = candidate words (bit i = word i of the slab)
//     w = word length | query length << 16
// and k_verify, launched right behind K2 on the same stream, runs the k <= 1
// verifiers on them (hamming_bounded / levenshtein_bounded,
// edit_distance.hpp:18-64) at high occupancy.  A record names its bytes
// directly, so the dependent chain is record -> (query bytes, word bytes) ->
// compare; the tables that turn offsets back into a query id and a sorted
// word position are only read for hits.  A warp takes 64 records at a time,
// lists their candidates in shared memory and verifies 64 per round, two per
// lane, all their bytes requested before any is compared; the next records
// are fetched a step ahead.  Hits leave as (query id << 32 | sorted word
// position) keys through the per-warp output chunks K4 reads.  The warps
// claim their records in stream order, which keeps the word bytes of the
// records in flight in L2; the kernel then is bound by instruction issue.
//
// The buffer has a fixed capacity per K2 launch.  Records reserved past its
// end are dropped and counted; k_verify raises the run's overflow flag and
// the host reruns the batch with a larger buffer, or with the tile plan cut
// into several K2 + K3 rounds that reuse the buffer (fpg_api.cu).
#pragma once

#include <cstdint>

namespace fpg {

struct VerifyParams {
    const uint32_t* q_start;    // per length: first sorted query position
    const uint64_t* q_bbase;    // per length: byte offset in the padded query blob
    const uint8_t* q_bytes;
    const uint32_t* q_ids;      // sorted position -> input query index
    const uint32_t* w_start;    // per length: first sorted word position
    const uint64_t* w_bbase;    // per length: byte offset in the padded word blob
    const uint8_t* w_bytes;
    unsigned long long* out;        // (query id << 32 | sorted word position) keys
    unsigned long long* out_count;  // key slots reserved (OutChunk)
    uint64_t out_cap;
    uint32_t* q_matches;        // per input query: matches (K4 segment sizes)
    int32_t k;
    int32_t pad_;
};

__device__ __forceinline__ int verify_stride(int len) { return len <= 16 ? 16 : (len + 15) & ~15; }

template <int NW>
__device__ __forceinline__ void load_words(const uint8_t* p, int stride, uint32_t (&r)[NW]) {
    const uint4 a = __ldg(reinterpret_cast<const uint4*>(p));
    r[0] = a.x; r[1] = a.y; r[2] = a.z; r[3] = a.w;
    if constexpr (NW == 8) {
        uint4 b = make_uint4(0, 0, 0, 0);
        if (stride > 16) b = __ldg(reinterpret_cast<const uint4*>(p) + 1);
        r[4] = b.x; r[5] = b.y; r[6] = b.z; r[7] = b.w;
    }
}

// hamming_bounded (edit_distance.hpp:18-27) as a test on register strings of
// equal length (zero padded): the bytes that differ are flagged in bit 7 of
// each byte and counted, at most k may differ.
template <int NW>
__device__ __forceinline__ bool hamming_regs(const uint32_t (&q)[NW], const uint32_t (&w)[NW], int k) {
    int cnt = 0;
#pragma unroll
    for (int i = 0; i < NW; ++i) {
        const uint32_t x = q[i] ^ w[i];
        cnt += __popc((((x & 0x7f7f7f7fu) + 0x7f7f7f7fu) | x) & 0x80808080u);
    }
    return cnt <= k;
}

// Warp-collective.  Every lane brings two records (z = 0: none); strings of
// up to 4 NW bytes are compared from registers, longer ones from memory.
// The 64 records' candidates (one per mask bit) are first listed in shared
// memory in lane order, so that every round verifies 64 of them, two per
// lane, whatever the lanes' own counts (a lane-private loop over its masks
// ran 2.9 rounds per 64 records on config 5 where the list needs 1.4).
// s_rec: the warp's 64 records, s_list: <= 2048 entries (record << 5 | bit).
// `pairs` accumulates the lane's candidate pairs (diagnostics).
template <int NW>
__device__ __forceinline__ void verify_records(const VerifyParams& V, uint4 ea, uint4 eb, OutChunk& oc, uint32_t& pairs,
                                               uint4* s_rec, uint16_t* s_list) {
    const int lane = threadIdx.x & 31;
    const uint32_t ca = (uint32_t)__popc(ea.z), cb = (uint32_t)__popc(eb.z);
    pairs += ca + cb;
    uint32_t incl = ca + cb;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const uint32_t v = __shfl_up_sync(0xffffffffu, incl, d);
        if (lane >= d) incl += v;
    }
    const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
    if (total == 0) return;
    __syncwarp();  // the previous call's readers are done with s_rec / s_list
    s_rec[lane] = ea;
    s_rec[32 + lane] = eb;
    {
        uint32_t rank = incl - (ca + cb);
        for (uint32_t mk = ea.z; mk; mk &= mk - 1) s_list[rank++] = (uint16_t)((lane << 5) | (__ffs(mk) - 1));
        for (uint32_t mk = eb.z; mk; mk &= mk - 1) s_list[rank++] = (uint16_t)(((32 + lane) << 5) | (__ffs(mk) - 1));
    }
    __syncwarp();
    for (uint32_t base = 0; base < total; base += 64) {
        // two candidates per lane and round: all their bytes are requested
        // before any is compared
        bool have[2];
        int len[2];                 // word length | query length << 16
        uint32_t qo[2], wo[2];      // byte offsets / 16 of the query and of the candidate word
        uint32_t qa[2][NW], bw[2][NW];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            const uint32_t idx = base + 32u * u + (uint32_t)lane;
            have[u] = idx < total;
            len[u] = 0;
            qo[u] = wo[u] = 0u;
#pragma unroll
            for (int c = 0; c < NW; ++c) qa[u][c] = bw[u][c] = 0u;
            if (have[u]) {
                const uint32_t e = s_list[idx];
                const uint4 r = s_rec[e >> 5];
                len[u] = (int)r.w;
                const int n = len[u] & 0xffff, m = len[u] >> 16;
                const int ws = verify_stride(n);
                qo[u] = r.x;
                wo[u] = r.y + (e & 31u) * (uint32_t)(ws >> 4);
                if ((m > n ? m : n) <= 4 * NW) {
                    load_words<NW>(V.q_bytes + 16ull * qo[u], verify_stride(m), qa[u]);
                    load_words<NW>(V.w_bytes + 16ull * wo[u], ws, bw[u]);
                }
            }
        }
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            if (u && base + 32u >= total) break;  // warp-uniform
            bool hit = false;
            const int n = len[u] & 0xffff, m = len[u] >> 16;
            if (have[u]) {
                if (m == n && n <= 4 * NW)
                    hit = hamming_regs<NW>(qa[u], bw[u], V.k);
                else if ((m > n ? m : n) <= 4 * NW)
                    hit = verify_regs<NW>(qa[u], bw[u], m, n, V.k);
                else
                    hit = verify_pair(V.q_bytes + 16ull * qo[u], m, verify_stride(m), V.w_bytes + 16ull * wo[u], n,
                                      verify_stride(n), V.k);
            }
            const uint32_t hb = __ballot_sync(0xffffffffu, hit);
            if (hb) {
                // offsets back to the sorted positions (hits only)
                uint32_t qid = 0, wpos = 0;
                if (hit) {
                    const uint32_t qs16 = (uint32_t)verify_stride(m) >> 4, ws16 = (uint32_t)verify_stride(n) >> 4;
                    const uint32_t qrel = qo[u] - (uint32_t)(V.q_bbase[m] >> 4), wrel = wo[u] - (uint32_t)(V.w_bbase[n] >> 4);
                    qid = V.q_ids[V.q_start[m] + (qs16 == 1 ? qrel : qrel / qs16)];
                    wpos = V.w_start[n] + (ws16 == 1 ? wrel : wrel / ws16);
                }
                const bool head = match_run_head(hit, qid, hb);
                const uint32_t heads = __ballot_sync(0xffffffffu, head);
                oc.emit(hb, hit, ((uint64_t)qid << 32) | wpos, V.out, V.out_cap, V.out_count);
                if (hit) count_match(V.q_matches, qid, hb, head, heads);
            }
        }
    }
}

constexpr int kVerifyThreads = 256;
constexpr int kVerifyChunk = 256;  // records a warp claims at a time

#ifndef FPG_K2_TU  // defined once, in fpg_api.cu
// n_records = records K2 reserved this round (may exceed cap: the excess was
// dropped; `overflow` tells the host, `peak` sizes its next attempt).
template <int NW>
__global__ void __launch_bounds__(kVerifyThreads, NW == 4 ? 4 : 3) k_verify(const __grid_constant__ VerifyParams V,
                                                           const uint4* __restrict__ records,
                                                           const unsigned long long* __restrict__ n_records,
                                                           uint64_t cap, unsigned long long* __restrict__ match_total,
                                                           unsigned long long* __restrict__ candidates,
                                                           unsigned long long* __restrict__ overflow,
                                                           unsigned long long* __restrict__ peak,
                                                           unsigned long long* __restrict__ cursor) {
    const uint64_t used = *n_records;
    const uint64_t n = used < cap ? used : cap;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        if (used > cap) *overflow = 1ull;
        if (used > *peak) *peak = used;  // rounds are stream-ordered: no race
    }
    const int lane = threadIdx.x & 31;
    OutChunk oc;
    uint32_t pairs = 0;
    const uint4 none = make_uint4(0u, 0u, 0u, 0u);
    constexpr uint64_t kNoBlock = ~0ull;
    __shared__ __align__(16) uint4 s_rec_all[kVerifyThreads / 32][64];
    __shared__ uint16_t s_list_all[kVerifyThreads / 32][64 * 32];
    uint4* s_rec = s_rec_all[threadIdx.x >> 5];
    uint16_t* s_list = s_list_all[threadIdx.x >> 5];
    // The warps claim chunks of kVerifyChunk records from a shared cursor, in
    // stream order, so that the records in flight on the whole GPU are one
    // window of the stream whatever the warps' speeds: records of one K2
    // moment concern one slab range, whose word bytes then stay in L2 (a
    // static, strided split lets the warps drift hundreds of MB apart).
    uint64_t chunk = kNoBlock;
    int sub = kVerifyChunk / 64;
    auto next_block = [&]() -> uint64_t {  // 64 records per warp and step
        if (sub == kVerifyChunk / 64) {
            unsigned long long c = 0;
            if (lane == 0) c = atomicAdd(cursor, 1ull);
            chunk = __shfl_sync(0xffffffffu, c, 0) * (uint64_t)kVerifyChunk;
            sub = 0;
        }
        if (chunk >= n) return kNoBlock;
        return chunk + 64u * (uint32_t)(sub++);
    };
    auto fetch = [&](uint64_t b, uint4& ea, uint4& eb) {  // streamed once
        ea = b + lane < n ? __ldcs(records + b + lane) : none;
        eb = b + 32 + lane < n ? __ldcs(records + b + 32 + lane) : none;
    };
    uint4 ea = none, eb = none;
    uint64_t cur = next_block();
    if (cur != kNoBlock) fetch(cur, ea, eb);
    while (cur != kNoBlock) {
        uint4 na = none, nb = none;
        const uint64_t nxt = next_block();  // fetched a step ahead
        if (nxt != kNoBlock) fetch(nxt, na, nb);
        verify_records<NW>(V, ea, eb, oc, pairs, s_rec, s_list);
        ea = na;
        eb = nb;
        cur = nxt;
    }
    oc.close(V.out, V.out_cap);
    if (lane == 0 && oc.real) atomicAdd(match_total, (unsigned long long)oc.real);
    pairs = __reduce_add_sync(0xffffffffu, pairs);
    if (lane == 0 && pairs) atomicAdd(candidates, (unsigned long long)pairs);
}
#endif

}  // namespace fpg
