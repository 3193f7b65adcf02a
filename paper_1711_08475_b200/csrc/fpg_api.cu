// fpg_api.cu -- C ABI (include/fpg.h) over the sm_100a kernels.
//
// Host runtime: per-device shards of the dictionary (contiguous input-order
// id ranges, dictionary.hpp:51-56 keeps input order), per-batch device
// scratch and streams, tile planning over length buckets, and the host-side
// CSR merge across shards.  No compute happens on the host: fingerprints,
// filtering, verification, ordering and CSR construction all run on the GPU;
// the host only counting-sorts query lengths, plans tiles from bucket
// counts, turns the per-query survivor counts into QueryStats and
// concatenates shard rows.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <thread>
#include <type_traits>
#include <unordered_map>
#include <map>
#include <vector>

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_segmented_sort.cuh>
#include <cub/device/device_select.cuh>
#include <thrust/iterator/counting_iterator.h>

#include "../../include/fpg.h"
#include "fpg_host.h"
#include "fpg_kernels.cuh"

namespace {

thread_local std::string g_last_error;
using fpg_host::Error;

template <class F>
int guarded(F&& f) {
    // drop a non-sticky error left by an earlier failed call on this thread
    // (e.g. cudaSetDevice on a bad ordinal), so it is not blamed on this one
    (void)cudaGetLastError();
    try {
        f();
        return FPG_OK;
    } catch (const Error& e) {
        g_last_error = e.what();
        return e.code;
    } catch (const std::bad_alloc&) {
        g_last_error = "host allocation failed";
        return FPG_ENOMEM;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return FPG_ECUDA;
    }
}

inline uint64_t cdiv(uint64_t a, uint64_t b) { return (a + b - 1) / b; }
// per-run device counters: key slots reserved, survivors, tile counter, verifier
// candidates, big segment flag, matches, pairs evaluated after the weight skip,
// segments listed for k_seg_sort_big, its bucket overflow flag, the exact
// path's tile counter and its pairs evaluated, candidate records reserved in
// the current K2 round, the candidate buffer's overflow flag, the largest
// per-round record count and K3's chunk cursor
constexpr int kNumCounters = 15;
constexpr unsigned kScatterBlocks = 148 * 4;  // grid-stride K4 scatter (the count is only known on the device)
inline int stride_of(int len) { return len <= 16 ? 16 : (len + 15) & ~15; }

// Device buffer that grows on demand (never shrinks), freed on destruction.
template <class T>
struct DBuf {
    T* p = nullptr;
    size_t cap = 0;  // elements
    int dev = -1;
    void reserve(size_t n) {
        if (n <= cap && p) return;
        release();
        size_t want = std::max<size_t>(n, 1);
        CK(cudaMalloc(&p, want * sizeof(T)));
        cap = want;
        CK(cudaGetDevice(&dev));
    }
    void release() {
        if (p) {
            int cur = -1;
            cudaGetDevice(&cur);
            if (dev >= 0 && cur != dev) cudaSetDevice(dev);
            cudaFree(p);
            if (dev >= 0 && cur != dev) cudaSetDevice(cur);
        }
        p = nullptr;
        cap = 0;
    }
    ~DBuf() { release(); }
    DBuf() = default;
    DBuf(const DBuf&) = delete;
    DBuf& operator=(const DBuf&) = delete;
};

// Pinned host buffer.
template <class T>
struct HBuf {
    T* p = nullptr;
    size_t cap = 0;
    void reserve(size_t n) {
        if (n <= cap && p) return;
        release();
        size_t want = std::max<size_t>(n, 1);
        CK(cudaMallocHost(&p, want * sizeof(T)));
        cap = want;
    }
    void release() {
        if (p) cudaFreeHost(p);
        p = nullptr;
        cap = 0;
    }
    ~HBuf() { release(); }
    HBuf() = default;
    HBuf(const HBuf&) = delete;
    HBuf& operator=(const HBuf&) = delete;
};

// Page-locked blocks for result arrays (fpg_result): a download writes the
// CSR straight into them (one D2H, no staging copy, no first-touch page
// faults), and fpg_result_free returns them here for the next result of a
// similar size.  Process-wide; idle blocks are capped at kPinnedIdleMax.
struct PinnedPool {
    static constexpr size_t kPinnedIdleMax = size_t(4) << 30;
    std::mutex mu;
    std::unordered_map<void*, size_t> owned;  // every block of the pool -> bytes
    std::multimap<size_t, void*> idle;
    size_t idle_bytes = 0;
    void* get(size_t bytes) {
        bytes = std::max<size_t>(bytes, 64);
        {
            std::lock_guard<std::mutex> lk(mu);
            auto it = idle.lower_bound(bytes);
            if (it != idle.end() && it->first <= 2 * bytes + (size_t(1) << 20)) {
                void* p = it->second;
                idle_bytes -= it->first;
                idle.erase(it);
                return p;
            }
        }
        void* p = nullptr;
        if (cudaHostAlloc(&p, bytes, cudaHostAllocPortable) != cudaSuccess || !p) {
            cudaGetLastError();
            throw std::bad_alloc();
        }
        std::lock_guard<std::mutex> lk(mu);
        owned[p] = bytes;
        return p;
    }
    // false: not a pool block (the caller frees it)
    bool put(void* p) {
        if (!p) return true;
        std::lock_guard<std::mutex> lk(mu);
        auto it = owned.find(p);
        if (it == owned.end()) return false;
        const size_t bytes = it->second;
        if (idle_bytes + bytes > kPinnedIdleMax) {
            owned.erase(it);
            cudaFreeHost(p);
        } else {
            idle.emplace(bytes, p);
            idle_bytes += bytes;
        }
        return true;
    }
};
PinnedPool& pinned_pool() {
    static PinnedPool* pool = new PinnedPool;  // never destroyed: results may outlive static teardown
    return *pool;
}

fpg::SchemeParams make_params(const fpg_scheme& s) {
    fpg::SchemeParams P;
    std::memset(&P, 0, sizeof(P));
    for (int c = 0; c < 256; ++c) P.slot[c] = P.sigbit[c] = -1;
    for (int i = 0; i < s.nletters; ++i) P.slot[s.letters[i]] = (int8_t)i;
    P.variant = s.variant;
    P.width = s.width;
    P.b = s.bits_per_count;
    P.p = s.bits_per_position;
    P.nletters = s.nletters;
    const int W = s.width;
    P.full = W == 64 ? ~0ull : ((1ull << W) - 1);
    if (s.variant == FPG_COUNT) {
        for (int q = 0; q < W / P.b; ++q) P.mask_fold |= 1ull << (W - P.b * (q + 1));
        P.onehot = (W == 16 && P.b == 2) ? 1 : 0;
    } else if (s.variant == FPG_POSITION) {
        P.slots = W / P.p;
        P.extra = W - P.slots * P.p;
        for (int q = 0; q < P.slots; ++q) P.mask_fold |= 1ull << (W - P.p * (q + 1));
        for (int q = 0; q < P.extra; ++q) P.mask_single |= 1ull << q;
    }
    return P;
}

int capacity(int32_t variant, int32_t width, int32_t b, int32_t p) {
    if (width != 16 && width != 32 && width != 64) return FPG_EINVAL;
    switch (variant) {
        case FPG_OCCURRENCE: return width;
        case FPG_OCCURRENCE_HALVED: return width / 2;
        case FPG_COUNT: return (b <= 0 || width % b) ? FPG_EINVAL : width / b;
        case FPG_POSITION: {
            if (p <= 0 || p > width) return FPG_EINVAL;
            const int slots = width / p;
            return slots + (width - slots * p);
        }
    }
    return FPG_EINVAL;
}

void validate(const fpg_scheme* s) {
    if (!s) throw Error(FPG_EINVAL, "null scheme");
    const int cap = capacity(s->variant, s->width, s->bits_per_count, s->bits_per_position);
    if (cap < 0) throw Error(FPG_EINVAL, "invalid scheme parameters (variant/width/b/p)");
    if (s->nletters != cap)
        throw Error(FPG_EINVAL, "scheme requires " + std::to_string(cap) + " letters, got " +
                                    std::to_string(s->nletters));
    bool seen[256] = {false};
    for (int i = 0; i < s->nletters; ++i) {
        if (seen[s->letters[i]]) throw Error(FPG_EINVAL, "LetterSet: duplicate symbol in letter set");
        seen[s->letters[i]] = true;
    }
}

bool supports(int variant, int metric) {
    return metric == FPG_HAMMING || variant == FPG_OCCURRENCE || variant == FPG_COUNT;
}

std::atomic<uint64_t> g_launches{0};  // per process; per-run counts are exact

// FPG_WSKIP=0 turns K2's weight window off (A/B runs)
const bool g_no_wskip = [] {
    const char* e = std::getenv("FPG_WSKIP");
    return e && e[0] == '0';
}();

const bool g_trace = [] {
    const char* e = std::getenv("FPG_TRACE");
    return e && e[0] == '1';
}();

double env_double(const char* name, double dflt) {
    const char* e = std::getenv(name);
    return e && *e ? std::atof(e) : dflt;
}  // approximate, per process; per-run counts are exact below

// The verifier's occurrence-signature pre-check (exact; see occurrence_sig)
// can be switched off with FPG_SIG_PRECHECK=0 to compare both paths.
const bool g_sig_precheck = [] {
    const char* e = std::getenv("FPG_SIG_PRECHECK");
    return !(e && e[0] == '0');
}();

enum BuildMode { kGenericDict = 0, kSliceDict = 1, kSliceQuery = 2 };

// Strings of one collection, length-bucketed on one device.
struct Collection {
    uint64_t n = 0;
    std::vector<uint32_t> count, start;  // per length [0, kMaxLen]
    std::vector<uint64_t> byte_base;
    uint64_t total_bytes = 0;
    int max_len = 0;
    DBuf<uint64_t> fp;   // reference-layout fingerprints (prints())
    DBuf<uint64_t> cmp;  // generic K2: comparison words (== fp, or the one-hot count-16 form)
    DBuf<uint32_t> sig;  // generic K2: occurrence signatures (verifier pre-check)
    DBuf<uint32_t> sigp; // bit-sliced K2: sig' codes (fpg_slice.cuh)
    DBuf<uint32_t> ids;
    DBuf<uint8_t> bytes;
    DBuf<uint32_t> d_start;
    DBuf<uint64_t> d_byte_base;
    // bit-sliced dictionary: per length slab ranges and plane offsets
    std::vector<uint32_t> slab_start;    // L1 + 1
    std::vector<uint64_t> plane_base;    // L1
    DBuf<uint32_t> planes;
    DBuf<uint32_t> wt;        // bit-sliced K2: group weights (fp_gweight) per sorted position
    DBuf<uint32_t> xc;        // position path: symbol codes of kXLen byte positions (kXBits each)
    DBuf<uint32_t> xplanes;   // position path planes (every bucket): the code planes
    std::vector<uint64_t> xplane_base;  // per length: u32 offset in xplanes
    DBuf<uint64_t> d_xplane_base;
    DBuf<uint2> slab_w;       // bit-sliced dictionary: group-weight box (min, max nibbles) per global slab
    DBuf<uint2> gbox;         // ... and per slab group (32 * SL slabs of a bucket)
    std::vector<uint32_t> group_start;  // L1 + 1: first global slab group of each bucket
    DBuf<uint32_t> d_group_start;
    DBuf<uint64_t> wkey_a, wkey_b;  // scratch: (length << 32 | group weights) sort keys
    DBuf<uint32_t> d_slab_start, d_count;
    DBuf<uint64_t> d_plane_base;
    // W = 16 dictionaries: fingerprint histogram per present length (+ one over
    // all lengths) and the XOR masks within F_D <= 2 (k_fp_stats): QueryStats
    // without survivor counters in K2
    DBuf<uint32_t> fph;        // [(nh + 1) * 65536]
    DBuf<int32_t> d_hslot;     // per length: histogram slot or -1
    DBuf<uint32_t> d_hfirst;   // per slot: first sorted position
    DBuf<uint16_t> d_hdelta;   // 0 first
    int nh = 0, n_hdelta = 0;
    // scratch (len_b = lengths in sorted order; kept for query collections)
    DBuf<uint16_t> len_a, len_b;
    DBuf<uint32_t> idx_a, idx_b;
    DBuf<uint32_t> hist;
    DBuf<uint8_t> cub_tmp;
    HBuf<uint32_t> h_hist;
    // construction profile (dictionary collections): per stage, CUDA-event
    // time on the build stream and algorithmic HBM bytes (reads + writes)
    std::vector<fpg_build_stage> stages;
    std::vector<cudaEvent_t> stage_ev;  // begin, end per stage (recorded around the launches only)
    void stage_mark(cudaStream_t st) {
        cudaEvent_t e;
        CK(cudaEventCreate(&e));
        CK(cudaEventRecord(e, st));
        stage_ev.push_back(e);
    }
    void stage_add(const char* name, double bytes) {  // after the stage's end mark
        fpg_build_stage g{};
        std::snprintf(g.name, sizeof(g.name), "%s", name);
        g.bytes = bytes;
        stages.push_back(g);
    }
    // after the build stream synchronised
    void stage_finish() {
        for (size_t i = 0; 2 * i + 1 < stage_ev.size() && i < stages.size(); ++i) {
            float ms = 0;
            CK(cudaEventElapsedTime(&ms, stage_ev[2 * i], stage_ev[2 * i + 1]));
            stages[i].ms = ms;
        }
        for (auto e : stage_ev) cudaEventDestroy(e);
        stage_ev.clear();
    }

    // Builds the bucketed layout of n strings already on the device.
    // Returns the number of kernel launches issued (ours, not CUB's).
    uint64_t build(const uint8_t* d_blob, const uint64_t* d_offs, uint64_t n_, const fpg::SchemeParams& P,
                   cudaStream_t st, BuildMode mode, int npt) {
        n = n_;
        const int L1 = fpg::kMaxLen + 1;
        count.assign(L1, 0);
        start.assign(L1, 0);
        byte_base.assign(L1, 0);
        uint64_t launches = 0;
        hist.reserve(L1 + 1);
        h_hist.reserve(L1 + 1);
        CK(cudaMemsetAsync(hist.p, 0, sizeof(uint32_t) * (L1 + 1), st));
        fp.reserve(n);
        if (mode == kGenericDict) {
            cmp.reserve(n);
            sig.reserve(n);
        } else {
            sigp.reserve(n);
        }
        ids.reserve(n);
        len_b.reserve(n);
        const bool prof = mode != kSliceQuery;
        stages.clear();
        if (n) {
            len_a.reserve(n); idx_a.reserve(n); idx_b.reserve(n);
            if (prof) stage_mark(st);
            fpg::k_lengths<<<(unsigned)std::min<uint64_t>(cdiv(n, 256), 148 * 8), 256, 0, st>>>(
                d_offs, n, len_a.p, idx_a.p, hist.p, hist.p + L1);
            CK(cudaGetLastError());
            ++launches;
            if (prof) {
                stage_mark(st);
                stage_add("k_lengths", 8.0 * (n + 1) + 6.0 * n);  // offsets in; lengths, identity ids out
            }
        }
        CK(cudaMemcpyAsync(h_hist.p, hist.p, sizeof(uint32_t) * (L1 + 1), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        if (h_hist.p[L1]) throw Error(FPG_EINVAL, "string longer than FPG_MAX_WORD_LEN");
        uint64_t pos = 0, bytes_pos = 0;
        max_len = 0;
        for (int L = 0; L < L1; ++L) {
            count[L] = h_hist.p[L];
            start[L] = (uint32_t)pos;
            byte_base[L] = bytes_pos;
            pos += count[L];
            bytes_pos += (uint64_t)count[L] * stride_of(L);
            if (count[L]) max_len = L;
        }
        total_bytes = bytes_pos;
        bytes.reserve(total_bytes);
        d_start.reserve(L1);
        d_byte_base.reserve(L1);
        CK(cudaMemcpyAsync(d_start.p, start.data(), sizeof(uint32_t) * L1, cudaMemcpyHostToDevice, st));
        CK(cudaMemcpyAsync(d_byte_base.p, byte_base.data(), sizeof(uint64_t) * L1, cudaMemcpyHostToDevice, st));
        if (!n) return launches;
        int end_bit = 1;
        while ((1 << end_bit) <= max_len) ++end_bit;
        uint64_t ends[2] = {0, 0};  // offsets[0], offsets[n]: the word bytes K1 reads
        CK(cudaMemcpyAsync(&ends[0], d_offs, sizeof(uint64_t), cudaMemcpyDeviceToHost, st));
        CK(cudaMemcpyAsync(&ends[1], d_offs + n, sizeof(uint64_t), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        const uint64_t blob_bytes = ends[1] - ends[0];
        size_t tmp = 0;
        const unsigned grid = (unsigned)cdiv(n, 256);
        if (mode == kSliceDict) {
            // stable sort by (length, group weights): inside a length bucket the
            // words are ordered by their group weights, so K2 warps see narrow
            // group-weight boxes
            wkey_a.reserve(n);
            wkey_b.reserve(n);
            if (prof) stage_mark(st);
#define FPG_KEYS(V) fpg::k_weight_keys<V><<<grid, 256, 0, st>>>(d_blob, d_offs, n, P, wkey_a.p)
            switch (P.variant) {
                case 0: FPG_KEYS(0); break;
                case 1: FPG_KEYS(1); break;
                case 2: FPG_KEYS(2); break;
                default: FPG_KEYS(3); break;
            }
#undef FPG_KEYS
            CK(cudaGetLastError());
            ++launches;
            if (prof) {
                stage_mark(st);
                // offsets and word bytes in, (length, group weights) keys out
                stage_add("k_weight_keys", 8.0 * (n + 1) + (double)blob_bytes + 8.0 * n);
            }
            CK(cub::DeviceRadixSort::SortPairs(nullptr, tmp, wkey_a.p, wkey_b.p, idx_a.p, idx_b.p, (int)n, 0,
                                               end_bit + 32, st));
            cub_tmp.reserve(tmp);
            if (prof) stage_mark(st);
            CK(cub::DeviceRadixSort::SortPairs(cub_tmp.p, tmp, wkey_a.p, wkey_b.p, idx_a.p, idx_b.p, (int)n, 0,
                                               end_bit + 32, st));
            wt.reserve(n);
        } else {
            CK(cub::DeviceRadixSort::SortPairs(nullptr, tmp, len_a.p, len_b.p, idx_a.p, idx_b.p, (int)n, 0,
                                               end_bit, st));
            cub_tmp.reserve(tmp);
            if (prof) stage_mark(st);
            CK(cub::DeviceRadixSort::SortPairs(cub_tmp.p, tmp, len_a.p, len_b.p, idx_a.p, idx_b.p, (int)n, 0,
                                               end_bit, st));
        }
        if (prof) {
            stage_mark(st);
            // CUB onesweep (library): one read + write of keys and values per 8-bit digit pass
            const int passes = ((mode == kSliceDict ? end_bit + 32 : end_bit) + 7) / 8;
            stage_add("cub_radix_sort", passes * 2.0 * (mode == kSliceDict ? 12.0 : 6.0) * n);
        }
        uint64_t* cmp_p = mode == kGenericDict ? cmp.p : nullptr;
        uint32_t* sig_p = mode == kGenericDict ? sig.p : nullptr;
        uint32_t* sigp_p = mode == kGenericDict ? nullptr : sigp.p;
        if (prof) stage_mark(st);
        uint32_t* xc_p = nullptr;
        if (mode == kSliceDict && P.xlen) {
            xc.reserve(n);
            xc_p = xc.p;
        }
#define FPG_BUILD(V) fpg::k_build<V><<<grid, 256, 0, st>>>(d_blob, d_offs, idx_b.p, n, d_start.p, d_byte_base.p, P, \
                                                           fp.p, cmp_p, sig_p, sigp_p, ids.p, bytes.p, nullptr,    \
                                                           nullptr, nullptr, 0, mode == kSliceDict ? wt.p : nullptr, xc_p)
        switch (P.variant) {
            case 0: FPG_BUILD(0); break;
            case 1: FPG_BUILD(1); break;
            case 2: FPG_BUILD(2); break;
            default: FPG_BUILD(3); break;
        }
#undef FPG_BUILD
        CK(cudaGetLastError());
        ++launches;
        if (prof) {
            stage_mark(st);
            // order, offsets and word bytes in; fingerprints, codes, ids, padded bytes (and weights) out
            const double out_w = mode == kSliceDict ? 8.0 + 4.0 + 4.0 + 4.0 : 8.0 + 8.0 + 4.0 + 4.0;
            stage_add("k_build", 4.0 * n + 8.0 * (n + 1) + (double)blob_bytes + out_w * n + (double)total_bytes);
        }
        // pre-check off: equal (zero) signatures pass every pair through
        if (mode == kGenericDict && !g_sig_precheck) CK(cudaMemsetAsync(sig.p, 0, n * sizeof(uint32_t), st));
        if (mode == kSliceDict) {
            slab_start.assign(L1 + 1, 0);
            plane_base.assign(L1, 0);
            uint64_t sl = 0, pb = 0;
            for (int L = 0; L < L1; ++L) {
                slab_start[L] = (uint32_t)sl;
                plane_base[L] = pb;
                const uint64_t ns = cdiv(count[L], 32);
                sl += ns;
                pb += cdiv(ns, 32) * 32 * (uint64_t)npt;  // whole rows of 32 slabs (fpg_slice.cuh layout)
            }
            slab_start[L1] = (uint32_t)sl;
            planes.reserve(pb);
            d_slab_start.reserve(L1 + 1);
            d_count.reserve(L1);
            d_plane_base.reserve(L1);
            CK(cudaMemcpyAsync(d_slab_start.p, slab_start.data(), sizeof(uint32_t) * (L1 + 1), cudaMemcpyHostToDevice, st));
            CK(cudaMemcpyAsync(d_count.p, count.data(), sizeof(uint32_t) * L1, cudaMemcpyHostToDevice, st));
            CK(cudaMemcpyAsync(d_plane_base.p, plane_base.data(), sizeof(uint64_t) * L1, cudaMemcpyHostToDevice, st));
            slab_w.reserve(sl);
            if (prof) stage_mark(st);
            fpg::k_planes<<<(unsigned)cdiv(sl, fpg::kPlanesSlabs), 32 * fpg::kPlanesSlabs, 0, st>>>(fp.p, sigp.p, wt.p, slab_w.p,
                                                                        d_slab_start.p, d_start.p,
                                                                        d_count.p, d_plane_base.p, L1, (uint32_t)sl,
                                                                        P.width, npt, planes.p);
            CK(cudaGetLastError());
            ++launches;
            if (prof) {
                stage_mark(st);
                // fingerprints, codes, weights in; planes and slab boxes out
                stage_add("k_planes", 16.0 * n + 4.0 * (double)pb + 8.0 * (double)sl);
            }
            // group boxes: the unit K2 warps claim is 32 * SL slabs
            const uint32_t gsl = (uint32_t)fpg::slice_group_slabs(npt);
            group_start.assign(L1 + 1, 0);
            uint32_t ng = 0;
            for (int L = 0; L < L1; ++L) {
                group_start[L] = ng;
                ng += (uint32_t)cdiv(count[L] ? cdiv(count[L], 32) : 0, gsl);
            }
            group_start[L1] = ng;
            gbox.reserve(std::max<uint32_t>(ng, 1));
            d_group_start.reserve(L1 + 1);
            CK(cudaMemcpyAsync(d_group_start.p, group_start.data(), sizeof(uint32_t) * (L1 + 1), cudaMemcpyHostToDevice, st));
            if (ng) {
                fpg::k_group_box<<<(unsigned)cdiv(ng, 256), 256, 0, st>>>(slab_w.p, d_slab_start.p, d_group_start.p, L1,
                                                                          ng, gsl, gbox.p);
                CK(cudaGetLastError());
                ++launches;
            }
            if (P.xlen) {
                // position-code planes (same kernel), every bucket: the symbol codes
                // of kXLen byte positions of each word (k_build: all positions of a
                // word of <= kXLen bytes, else kXLen positions spread over the word)
                const int xnpt = fpg::kXBits * fpg::kXLen;  // code planes only (QueryStats come from the histograms)
                xplane_base.assign(L1, 0);
                uint64_t xb = 0;
                for (int L = 0; L < L1; ++L) {
                    xplane_base[L] = xb;
                    xb += cdiv(cdiv(count[L], 32), 32) * 32 * (uint64_t)xnpt;
                }
                const uint32_t xsl = slab_start[L1];
                if (xsl) {
                    xplanes.reserve(xb);
                    d_xplane_base.reserve(L1);
                    CK(cudaMemcpyAsync(d_xplane_base.p, xplane_base.data(), sizeof(uint64_t) * L1, cudaMemcpyHostToDevice,
                                       st));
                    fpg::k_planes<<<(unsigned)cdiv(xsl, fpg::kPlanesSlabs), 32 * fpg::kPlanesSlabs, 0, st>>>(
                        fp.p, xc.p, nullptr, nullptr, d_slab_start.p, d_start.p, d_count.p, d_xplane_base.p, L1, xsl, 0,
                        xnpt, xplanes.p);
                    CK(cudaGetLastError());
                    ++launches;
                }
            }
            launches += build_fp_hist(P, st);
        }
        return launches;
    }

    // Fingerprint histograms for QueryStats (fpg_kernels.cuh, k_fp_stats): 16-bit
    // schemes with at most kMaxHistLengths present lengths.
    static constexpr int kMaxHistLengths = 256;
    uint64_t build_fp_hist(const fpg::SchemeParams& P, cudaStream_t st) {
        nh = 0;
        if (P.width != 16 || !n) return 0;
        const int L1 = fpg::kMaxLen + 1;
        std::vector<int32_t> hslot(L1, -1);
        std::vector<uint32_t> hfirst;
        for (int L = 0; L < L1; ++L)
            if (count[L]) {
                hslot[L] = (int32_t)hfirst.size();
                hfirst.push_back(start[L]);
            }
        if ((int)hfirst.size() > kMaxHistLengths) return 0;
        nh = (int)hfirst.size();
        // XOR masks touching at most two fields (F_D <= 2), 0 first
        std::vector<uint16_t> fmask;  // one bit mask per field
        const int fw = P.variant == FPG_COUNT ? P.b : P.variant == FPG_POSITION ? P.p : 1;
        const int extra = P.variant == FPG_POSITION ? P.extra : 0;
        const int nf = (16 - extra) / fw;
        for (int f = 0; f < nf; ++f) fmask.push_back((uint16_t)(((1u << fw) - 1u) << (16 - fw * (f + 1))));
        for (int e = 0; e < extra; ++e) fmask.push_back((uint16_t)(1u << e));
        std::vector<uint16_t> deltas{0};
        auto values = [&](uint16_t m, auto&& f) {  // every non-zero value inside mask m
            for (uint32_t v = m; v; v = (v - 1) & m) f((uint16_t)v);
        };
        for (size_t a = 0; a < fmask.size(); ++a)
            values(fmask[a], [&](uint16_t va) {
                deltas.push_back(va);
                for (size_t b = a + 1; b < fmask.size(); ++b) values(fmask[b], [&](uint16_t vb) { deltas.push_back(va | vb); });
            });
        n_hdelta = (int)deltas.size();
        fph.reserve((size_t)(nh + 1) * 65536);
        d_hslot.reserve(L1);
        d_hfirst.reserve(nh);
        d_hdelta.reserve(deltas.size());
        CK(cudaMemsetAsync(fph.p, 0, (size_t)(nh + 1) * 65536 * sizeof(uint32_t), st));
        CK(cudaMemcpyAsync(d_hslot.p, hslot.data(), L1 * sizeof(int32_t), cudaMemcpyHostToDevice, st));
        CK(cudaMemcpyAsync(d_hfirst.p, hfirst.data(), nh * sizeof(uint32_t), cudaMemcpyHostToDevice, st));
        CK(cudaMemcpyAsync(d_hdelta.p, deltas.data(), deltas.size() * sizeof(uint16_t), cudaMemcpyHostToDevice, st));
        fpg::k_fp_hist<<<(unsigned)cdiv(n, 256), 256, 0, st>>>(fp.p, n, d_hfirst.p, nh, fph.p);
        CK(cudaGetLastError());
        CK(cudaStreamSynchronize(st));  // the host vectors above go out of scope
        return 1;
    }

    void drop_scratch() {
        len_a.release(); len_b.release(); idx_a.release(); idx_b.release(); cub_tmp.release();
        wkey_a.release(); wkey_b.release();
    }

    // Query collection whose length order and bucket tables were built on the
    // host at upload (counting sort, fpg_batch_upload): one K1 launch, which
    // also zeroes the per-query survivor counts and the run counters.
    uint64_t build_sorted(const uint8_t* d_blob, const uint64_t* d_offs, const uint32_t* d_order,
                          const fpg::SchemeParams& P, cudaStream_t st, BuildMode mode, uint32_t* zero_by_id,
                          unsigned long long* zero64, int nzero64) {
        fp.reserve(n);
        if (mode == kGenericDict) {
            cmp.reserve(n);
            sig.reserve(n);
        } else {
            sigp.reserve(n);
        }
        ids.reserve(n);
        len_b.reserve(n);
        bytes.reserve(total_bytes);
        uint64_t* cmp_p = mode == kGenericDict ? cmp.p : nullptr;
        uint32_t* sig_p = mode == kGenericDict ? sig.p : nullptr;
        uint32_t* sigp_p = mode == kGenericDict ? nullptr : sigp.p;
        uint32_t* wt_p = nullptr;
        uint32_t* xc_p = nullptr;
        if (mode == kSliceQuery) {
            wt.reserve(n);
            wt_p = wt.p;
            if (P.xlen) {
                xc.reserve(n);
                xc_p = xc.p;
            }
        }
        const unsigned grid = (unsigned)std::max<uint64_t>(1, cdiv(n, 256));
#define FPG_BUILD(V) fpg::k_build<V><<<grid, 256, 0, st>>>(d_blob, d_offs, d_order, n, d_start.p, d_byte_base.p, P, \
                                                           fp.p, cmp_p, sig_p, sigp_p, ids.p, bytes.p, len_b.p,  \
                                                           zero_by_id, zero64, nzero64, wt_p, xc_p)
        switch (P.variant) {
            case 0: FPG_BUILD(0); break;
            case 1: FPG_BUILD(1); break;
            case 2: FPG_BUILD(2); break;
            default: FPG_BUILD(3); break;
        }
#undef FPG_BUILD
        CK(cudaGetLastError());
        if (mode == kGenericDict && !g_sig_precheck && n) CK(cudaMemsetAsync(sig.p, 0, n * sizeof(uint32_t), st));
        return 1;
    }
};

struct Shard {
    int device = 0;
    cudaStream_t stream = nullptr;
    uint64_t base = 0, n = 0;  // input index range [base, base + n)
    Collection dict;
    DBuf<uint8_t> blob;        // construction staging
    DBuf<uint64_t> offs;
    DBuf<unsigned long long> d_hist;
    HBuf<unsigned long long> h_hist;
};

}  // namespace

struct fpg_dict {
    fpg_scheme scheme;
    fpg::SchemeParams params;
    bool slice = false;     // bit-sliced K2 (fpg_slice.cuh); else the generic k_scan
    int npt = 0;            // planes per slab: W + sig' fields
    uint64_t n = 0, id_base = 0;
    std::vector<std::unique_ptr<Shard>> shards;
    std::vector<uint64_t> len_count;  // whole-dictionary bucket counts (all shards)
    double build_seconds = 0;
    std::mutex cache_mu;              // guards `pool`
    std::vector<fpg_batch*> pool;     // idle scratch batches of fpg_query_batch (one per concurrent caller)
    std::atomic<int> live_batches{0}; // fpg_batch_create handles not yet destroyed (they use the shards)
    ~fpg_dict();
};

namespace {

struct ShardBatch {
    Shard* sh = nullptr;
    cudaStream_t stream = nullptr;  // per batch: concurrent batches of one dictionary overlap
    DBuf<uint8_t> qblob;
    DBuf<uint64_t> qoffs;
    DBuf<uint32_t> qorder;
    Collection queries;
    DBuf<fpg::Tile> tiles;
    DBuf<fpg::SliceTile> stiles, stiles_x;
    std::vector<fpg::Tile> plan;
    std::vector<fpg::SliceTile> splan, splan_x;  // bit-sliced tiles; those of the exact path
    bool plan_valid = false;
    bool plan_small = false;  // the plan's tiles were made smaller than the full shape (few tiles per CTA)
    std::vector<uint32_t> plan_qcount;  // query length histogram the plan was built for
    fpg_query_options plan_opts{};
    DBuf<unsigned long long> out;
    DBuf<unsigned long long> counters;  // [0] out_count, [1] survivors_total, [2] tile counter
    DBuf<uint32_t> qsurv;
    DBuf<uint64_t> offsets;
    DBuf<uint32_t> ids, ids2;
    DBuf<uint32_t> big_list;  // K4: queries with more than kSegMax matches
    const uint32_t* ids_out = nullptr;  // sorted word ids of the last run (ids or ids2)
    DBuf<uint8_t> cub_tmp;
    HBuf<unsigned long long> h_counters;
    HBuf<uint64_t> h_offsets;
    HBuf<uint32_t> h_ids, h_qsurv;
    cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
    uint64_t total = 0, executed = 0, survivors = 0, candidates = 0, scanned = 0, scanned_x = 0, launches = 0;
    double run_ms = 0, filter_ms = 0, verify_ms = 0, plan_ms = 0;
    uint64_t out_cap = 1 << 20;
    // K2 -> K3 candidate records (fpg_verify.cuh): capacity per round (0: sized
    // from the plan at first use) and the K2 + K3 rounds the tile plan is cut
    // into when one round's records would not fit
    DBuf<uint4> cand;
    uint64_t cand_cap = 0, cand_records = 0, cand_fail = 0;
    uint32_t cand_rounds = 1;
    std::vector<cudaEvent_t> ev_k3;  // per round: before / after k_verify
};

}  // namespace

struct fpg_batch {
    fpg_dict* dict = nullptr;
    uint64_t nq = 0;
    std::vector<uint32_t> qlen;  // host copy of query lengths (stats bookkeeping)
    // length buckets of the queries (host counting sort at upload)
    std::vector<uint32_t> qcount, qstart;
    std::vector<uint64_t> qbbase;
    int qmax_len = 0;
    uint64_t qtotal_bytes = 0;
    HBuf<uint32_t> h_order, h_start;
    HBuf<uint64_t> h_bbase;
    std::vector<std::unique_ptr<ShardBatch>> sb;
    fpg_query_options opt{};
    bool uploaded = false;  // a batch of queries is on the devices
    bool ran = false;       // the last run succeeded (download is valid)
    bool external = false;  // created by fpg_batch_create (counted in dict->live_batches)
    double upload_ms = 0, download_ms = 0, assemble_ms = 0;  // host-side times of the last calls
    ~fpg_batch() {
        for (auto& s : sb) {
            cudaSetDevice(s->sh->device);
            for (auto e : s->ev)
                if (e) cudaEventDestroy(e);
            for (auto e : s->ev_k3)
                if (e) cudaEventDestroy(e);
            if (s->stream) cudaStreamDestroy(s->stream);
        }
    }
};

fpg_dict::~fpg_dict() {
    for (fpg_batch* b : pool) delete b;
    for (auto& s : shards) {
        cudaSetDevice(s->device);
        if (s->stream) cudaStreamDestroy(s->stream);
    }
}

namespace {

// Host-side assembly of large results in parallel: [0, n) cut into one range
// per thread (at least `grain` items each, up to the host's cores).  The
// threads also take the first-touch page faults of freshly allocated output.
template <class F>
void parallel_ranges(uint64_t n, uint64_t grain, F&& f) {
    static const unsigned hw = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
    const uint64_t t = std::max<uint64_t>(1, std::min<uint64_t>(hw, n / std::max<uint64_t>(grain, 1)));
    if (t == 1) {
        f(uint64_t(0), n);
        return;
    }
    std::vector<std::thread> th;
    for (uint64_t i = 0; i < t; ++i) th.emplace_back([&, i] { f(n * i / t, n * (i + 1) / t); });
    for (auto& x : th) x.join();
}

template <class F>
void for_each_shard(size_t n, F&& f) {
    if (n == 1) {
        f(0);
        return;
    }
    std::vector<std::thread> th;
    std::vector<std::string> errs(n);
    std::vector<int> codes(n, 0);
    for (size_t i = 0; i < n; ++i)
        th.emplace_back([&, i] {
            try {
                f(i);
            } catch (const Error& e) {
                errs[i] = e.what();
                codes[i] = e.code;
            } catch (const std::exception& e) {
                errs[i] = e.what();
                codes[i] = FPG_ECUDA;
            }
        });
    for (auto& t : th) t.join();
    for (size_t i = 0; i < n; ++i)
        if (codes[i]) throw Error(codes[i], "shard " + std::to_string(i) + ": " + errs[i]);
}

// Distance form per scheme: plain popcount (occurrence, halved, one-hot
// count-16), compile-time folds for count b=2/4 and position p=3, else the
// generic runtime fold.
int dist_kind(const fpg::SchemeParams& S, bool onehot) {
    if (S.variant == FPG_OCCURRENCE || S.variant == FPG_OCCURRENCE_HALVED || onehot) return fpg::kPopc;
    if (S.variant == FPG_COUNT) return S.b == 2 ? fpg::kFold2 : S.b == 4 ? fpg::kFold4 : fpg::kGeneric;
    return S.p == 3 ? fpg::kPos3 : fpg::kGeneric;
}

void dispatch_scan(const fpg::SchemeParams& S, bool onehot, bool stats, const fpg::Tile* tiles, uint32_t ntiles,
                   const fpg::ScanParams& P, cudaStream_t st, int device) {
    fpg_host::dispatch_scan(dist_kind(S, onehot), S.width, stats, tiles, ntiles, P, st, device);
}

// Field width of the scheme's multi-bit fields (1 for occurrence / halved).
int field_width_of(const fpg_scheme& s) {
    if (s.variant == FPG_COUNT) return s.bits_per_count;
    if (s.variant == FPG_POSITION) return s.bits_per_position;
    return 1;
}

bool slice_supported(const fpg_scheme& s) {
    const int fw = field_width_of(s);
    return fw >= 1 && fw <= 4;
}

void dispatch_slice(const fpg_scheme& sc, int nsig, const fpg::SliceTile* tiles, uint32_t ntiles,
                    const fpg::SliceParams& P, cudaStream_t st, int device) {
    const int fw = field_width_of(sc);
    if (sc.width == 16) fpg_host::dispatch_slice_16(fw, nsig, tiles, ntiles, P, st, device);
    else if (sc.width == 32) fpg_host::dispatch_slice_32(fw, nsig, tiles, ntiles, P, st, device);
    else fpg_host::dispatch_slice_64(fw, nsig, tiles, ntiles, P, st, device);
}

bool compatible(int metric, int k, int lq, int lw) {
    if (metric == FPG_HAMMING) return lq == lw;
    return std::abs(lq - lw) <= k;
}

// Plans tiles, scans, orders matches into a CSR on the shard's device.
void run_shard(fpg_dict* D, fpg_batch* B, ShardBatch& S, const fpg_query_options& o) {
    Shard& sh = *S.sh;
    CK(cudaSetDevice(sh.device));
    cudaStream_t st = S.stream;
    for (auto& e : S.ev)
        if (!e) CK(cudaEventCreate(&e));
    S.launches = 0;
    CK(cudaEventRecord(S.ev[0], st));
    const uint64_t nq = B->nq;
    // K1 on the queries (pattern fingerprint inside query time, dictionary.hpp:84)
    S.qsurv.reserve(2 * nq);  // [0, nq): fingerprint survivors, [nq, 2 nq): matches
    S.counters.reserve(kNumCounters);
    S.h_counters.reserve(kNumCounters);
    S.launches += S.queries.build_sorted(S.qblob.p, S.qoffs.p, S.qorder.p, D->params, st,
                                         D->slice ? kSliceQuery : kGenericDict, S.qsurv.p, S.counters.p,
                                         kNumCounters);
    const Collection& Q = S.queries;
    const Collection& W = sh.dict;
    uint64_t executed = 0;
    std::vector<fpg::Tile>& plan = S.plan;
    std::vector<fpg::SliceTile>& splan = S.splan;
    std::vector<fpg::SliceTile>& splan_x = S.splan_x;
    // QueryStats::verified from the fingerprint histograms instead of K2's
    // survivor counters (W = 16 dictionaries, k <= 1; FPG_HIST_STATS=0: A/B)
    const bool hist_on = env_double("FPG_HIST_STATS", 1.0) != 0.0;  // read per run: tests switch it
    const bool ext_stats = hist_on && D->slice && o.k <= 1 && W.nh > 0 && o.want_stats && o.use_filter && !o.exhaustive &&
                           supports(D->scheme.variant, o.metric);
    const bool count_only_pass =
        !ext_stats && o.want_stats && o.use_filter && o.metric == FPG_LEVENSHTEIN && !o.length_prefilter;
    // exact Hamming path for the words of <= kXLen bytes (fpg_slice.cuh, X);
    // its kernel holds no scheme planes, so it needs the stats to come from
    // the histograms (or not to be wanted)
    static const bool exact_on = env_double("FPG_EXACT", 1.0) != 0.0;
    const bool xpath = exact_on && D->params.xlen && o.metric == FPG_HAMMING && o.k <= 1 && !o.exhaustive &&
                       o.use_filter && (ext_stats || !o.want_stats);
    // The tile plan depends only on the batch's length histogram and the
    // options: it is built (and uploaded) once and reused by later runs and
    // by later batches with the same histogram.
    // the bit-sliced K2 covers k <= 1; larger k runs the generic per-pair
    // kernel (POPC filter, banded verifier) on the same collections
    const bool use_slice = D->slice && o.k <= 1;
    const bool from_slice = D->slice && !use_slice;  // generic kernel over bit-sliced collections
    const bool replan = !S.plan_valid || std::memcmp(&S.plan_opts, &o, sizeof(o)) != 0;
    const auto plan_t0 = std::chrono::steady_clock::now();
    if (!replan) {
        executed = S.executed;
    } else if (use_slice) {
        splan.clear();
        splan_x.clear();
        // Tile plan: per word length lw, the compatible query lengths form one
        // contiguous range of the length-sorted queries (Hamming / k = 0:
        // lw; Levenshtein k = 1: lw - 1 .. lw + 1, edit_distance.hpp:38-39).
        // Tiles = (<= kSliceMaxSlabs slabs) x (<= kSliceQ queries), largest first,
        // handed out by an atomic counter.
        const int L1 = fpg::kMaxLen + 1;
        // Tile shape: 128 queries x 256 slab groups (the warps claim the tile's
        // groups dynamically, so one tile's query masks serve many groups),
        // made smaller (slabs down to two groups per warp, queries down to 32,
        // slabs down to one group per warp, queries down to 16, then slabs down
        // to one group) while the batch would give fewer than ~4 tiles per
        // resident CTA.
        const uint32_t grp = (uint32_t)fpg::slice_group_slabs(D->npt);
        // FPG_TILE_GROUPS: slab groups per full tile (A/B runs); 256 = 32 per
        // warp, so the end-of-tile barrier waits on a small share of the tile
        // (config 5 K2: 64 groups 107.4 ms, 128 103.1, 256 101.4, 512 101.2)
        static const uint32_t tile_groups = (uint32_t)env_double("FPG_TILE_GROUPS", 256.0);
        uint32_t per = tile_groups * grp, qchunk = fpg::kSliceQ;
        int sms = 148;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, sh.device);
        {
            const uint64_t target = (uint64_t)sms * 2 * 4;
            auto count_tiles = [&]() {
                uint64_t c = 0;
                for (int lw = 0; lw <= W.max_len; ++lw) {
                    if (!W.count[lw]) continue;
                    const int span = (o.metric == FPG_HAMMING) ? 0 : o.k;
                    const int lo = std::max(0, lw - span), hi = std::min(L1 - 1, lw + span);
                    c += cdiv(Q.start[hi] + Q.count[hi] - Q.start[lo], qchunk) * cdiv(cdiv(W.count[lw], 32), per);
                }
                return c;
            };
            const uint32_t w8 = (uint32_t)fpg::kSliceWarps * grp;
            // FPG_TILE_GPW / FPG_TILE_Q: groups per warp and queries kept by the
            // first two shrink stages (A/B runs)
            static const uint32_t gpw = (uint32_t)env_double("FPG_TILE_GPW", 2.0);
            static const uint32_t q1 = (uint32_t)env_double("FPG_TILE_Q", 32.0);
            S.plan_small = count_tiles() < target;
            while (count_tiles() < target && (qchunk > 16 || per > grp)) {
                if (per > gpw * w8) per >>= 1;                 // down to gpw groups per warp
                else if (qchunk > q1) qchunk >>= 1;            // then q1 queries
                else if (per > w8) per >>= 1;                  // then 1 group per warp
                else if (qchunk > 16) qchunk >>= 1;
                else per >>= 1;
            }
        }
        auto add = [&](int lw, uint32_t qb, uint32_t qe, bool count_only) {
            const uint32_t ns = (uint32_t)cdiv(W.count[lw], 32);
            // slab range outer, query chunks inner: the tiles running at the same
            // time share one slab range, so its planes and the word bytes K3
            // reads for its candidates stay in L2
            for (uint32_t s0 = 0; s0 < ns; s0 += per)
                for (uint32_t q0 = qb; q0 < qe; q0 += qchunk) {
                    fpg::SliceTile t{};
                    t.slab_begin = s0;
                    t.n_slabs = std::min(per, ns - s0);
                    t.q_begin = q0;
                    t.q_count = std::min<uint32_t>(qchunk, qe - q0);
                    t.plane_base = W.plane_base[lw];
                    t.w_bytes = W.byte_base[lw];
                    t.ns = ns;
                    t.w_start = W.start[lw];
                    t.w_count = W.count[lw];
                    t.w_len = (uint16_t)lw;
                    t.w_stride = (uint16_t)stride_of(lw);
                    t.count_only = count_only ? 1u : 0u;
                    t.slab_g0 = W.slab_start[lw];
                    t.gbox_base = W.group_start[lw] + s0 / grp;
                    const bool xt = xpath && !count_only;  // every length: exact up to kXLen bytes, a position filter beyond
                    if (xt) t.plane_base = W.xplane_base[lw];
                    (xt ? splan_x : splan).push_back(t);
                }
        };
        for (int lw = 0; lw <= W.max_len; ++lw) {
            if (!W.count[lw]) continue;
            const int span = (o.metric == FPG_HAMMING) ? 0 : o.k;
            const int lo = std::max(0, lw - span), hi = std::min(L1 - 1, lw + span);
            const uint32_t qb = Q.start[lo], qe = Q.start[hi] + Q.count[hi];
            executed += (uint64_t)(qe - qb) * W.count[lw];
            add(lw, qb, qe, false);
            if (count_only_pass) {
                add(lw, 0, qb, true);
                add(lw, qe, (uint32_t)nq, true);
            }
        }
        // Largest tiles first; the tail of the schedule is cut into 32- and
        // 16-query tiles so the dynamically scheduled grid drains evenly.  A
        // small plan cuts everything after FPG_TAIL_A / FPG_TAIL_B of its
        // work; a large one only about its last 4 tiles per resident CTA
        // (small tiles cost a slab-group load per few queries: config 5 has
        // ~6e5 tiles and needs no cutting before its very end).
        auto cost = [](const fpg::SliceTile& x) { return (uint64_t)x.q_count * x.n_slabs; };
        static const double env_a = env_double("FPG_TAIL_A", 0.35), env_b = env_double("FPG_TAIL_B", 0.85);
        // each plan (one K2 launch) sorted largest first, its tail cut finer
        auto finish_plan = [&](std::vector<fpg::SliceTile>& pl, DBuf<fpg::SliceTile>& dev) {
            std::stable_sort(pl.begin(), pl.end(),
                             [&](const fpg::SliceTile& x, const fpg::SliceTile& y) { return cost(x) > cost(y); });
            uint64_t work = 0, acc = 0;
            for (const auto& t : pl) work += cost(t);
            std::vector<fpg::SliceTile> fine;
            fine.reserve(pl.size() + pl.size() / 2);
            const double tail_f = std::min(1.0, 4.0 * 2 * sms / std::max<double>(1.0, (double)pl.size()));
            const double tail_a = 1.0 - (1.0 - env_a) * tail_f, tail_b = 1.0 - (1.0 - env_b) * tail_f;
            for (const auto& t : pl) {
                acc += cost(t);
                const uint32_t sub = acc <= tail_a * work ? t.q_count : acc <= tail_b * work ? 32u : 16u;
                if (t.q_count <= sub) {
                    fine.push_back(t);
                    continue;
                }
                for (uint32_t q0 = 0; q0 < t.q_count; q0 += sub) {
                    fpg::SliceTile u = t;
                    u.q_begin = t.q_begin + q0;
                    u.q_count = std::min<uint32_t>(sub, t.q_count - q0);
                    fine.push_back(u);
                }
            }
            pl.swap(fine);
            dev.reserve(pl.size());
            if (!pl.empty())
                CK(cudaMemcpyAsync(dev.p, pl.data(), pl.size() * sizeof(fpg::SliceTile), cudaMemcpyHostToDevice, st));
        };
        // a small exact share does not pay for its own launch (latency-bound
        // batches): those tiles go back to the sig' path
        // (FPG_EXACT_MIN: pair threshold, read per plan so tests can force the path)
        uint64_t x_pairs = 0;
        for (const auto& t : splan_x) x_pairs += (uint64_t)t.q_count * t.n_slabs * 32u;
        if ((double)x_pairs < env_double("FPG_EXACT_MIN", 67108864.0)) {
            for (auto t : splan_x) {
                t.plane_base = W.plane_base[t.w_len];
                splan.push_back(t);
            }
            splan_x.clear();
        }
        finish_plan(splan, S.stiles);
        finish_plan(splan_x, S.stiles_x);
    } else {
        // Generic k_scan: one tile per (query length, word length) bucket pair block.
        plan.clear();
        for (int lq = 0; lq <= Q.max_len; ++lq) {
            if (!Q.count[lq]) continue;
            for (int lw = 0; lw <= W.max_len; ++lw) {
                if (!W.count[lw]) continue;
                const bool comp = compatible(o.metric, o.k, lq, lw);
                if (!comp && !count_only_pass) continue;
                if (comp) executed += (uint64_t)Q.count[lq] * W.count[lw];
                for (uint32_t q0 = 0; q0 < Q.count[lq]; q0 += fpg::kTileQueries) {
                    for (uint32_t w0 = 0; w0 < W.count[lw]; w0 += fpg::kTileWords) {
                        fpg::Tile t{};
                        t.q_begin = Q.start[lq] + q0;
                        t.q_count = std::min<uint32_t>(fpg::kTileQueries, Q.count[lq] - q0);
                        t.w_begin = W.start[lw] + w0;
                        t.w_count = std::min<uint32_t>(fpg::kTileWords, W.count[lw] - w0);
                        t.q_bytes = Q.byte_base[lq] + (uint64_t)q0 * stride_of(lq);
                        t.w_bytes = W.byte_base[lw] + (uint64_t)w0 * stride_of(lw);
                        t.q_len = (uint16_t)lq;
                        t.w_len = (uint16_t)lw;
                        t.q_stride = (uint16_t)stride_of(lq);
                        t.w_stride = (uint16_t)stride_of(lw);
                        t.count_only = comp ? 0u : 1u;
                        plan.push_back(t);
                    }
                }
            }
        }
        S.tiles.reserve(plan.size());
        if (!plan.empty())
            CK(cudaMemcpyAsync(S.tiles.p, plan.data(), plan.size() * sizeof(fpg::Tile), cudaMemcpyHostToDevice, st));
    }
    S.executed = executed;
    S.plan_valid = true;
    S.plan_opts = o;
    // host time of building (and queueing the upload of) a fresh tile plan;
    // later runs with the same length histogram and options reuse it
    if (replan) S.plan_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - plan_t0).count();

    fpg::ScanParams P{};
    fpg::SliceParams SP{};
    fpg::VerifyParams VP{};
    if (use_slice) {
        SP.planes = W.planes.p;
        SP.q_fp = Q.fp.p;
        SP.q_sigp = Q.sigp.p;
        SP.q_ids = Q.ids.p;
        SP.q_len = Q.len_b.p;
        SP.q_start = Q.d_start.p;
        SP.q_bbase = Q.d_byte_base.p;
        SP.q_survivors = S.qsurv.p;
        SP.survivors_total = S.counters.p + 1;
        SP.tile_counter = reinterpret_cast<unsigned int*>(S.counters.p + 2);
        SP.k = o.k;
        SP.stats = (o.want_stats && o.use_filter && !ext_stats) ? 1 : 0;
        SP.use_fp = supports(D->scheme.variant, o.metric) && !o.exhaustive ? 1 : 0;
        SP.exhaustive = o.exhaustive ? 1 : 0;
        SP.wskip = SP.use_fp && !o.exhaustive && !g_no_wskip ? 1 : 0;
        SP.q_weight = Q.wt.p;
        SP.slab_w = W.slab_w.p;
        SP.gbox = W.gbox.p;
        SP.scanned = S.counters.p + 6;
        static const int drop = (int)env_double("FPG_DROP_CANDIDATES", 0.0);
        SP.drop_candidates = drop;
        SP.cand_count = S.counters.p + 11;
        // K3 (k_verify): everything it needs to resolve a candidate record
        VP.q_start = Q.d_start.p;
        VP.q_bbase = Q.d_byte_base.p;
        VP.q_bytes = Q.bytes.p;
        VP.q_ids = Q.ids.p;
        VP.w_start = W.d_start.p;
        VP.w_bbase = W.d_byte_base.p;
        VP.w_bytes = W.bytes.p;
        VP.out_count = S.counters.p;
        VP.q_matches = S.qsurv.p + nq;
        VP.k = o.k;
    } else {
        // comparison words: the reference-layout fingerprints when the
        // collections were built for k_slice (no one-hot form, no signatures)
        const bool onehot = D->params.onehot && !from_slice;
        P.q_fp = from_slice ? Q.fp.p : Q.cmp.p;
        P.w_fp = from_slice ? W.fp.p : W.cmp.p;
        P.q_bytes = Q.bytes.p;
        P.q_ids = Q.ids.p;
        P.q_sig = Q.sig.p;
        P.w_sig = W.sig.p;
        P.sig_on = (!from_slice && o.k <= 1) ? 1 : 0;
        P.lev = o.metric == FPG_LEVENSHTEIN ? 1 : 0;
        P.w_bytes = W.bytes.p;
        P.w_ids = W.ids.p;
        P.id_base = D->id_base + sh.base;
        P.q_survivors = S.qsurv.p;
        P.out_count = S.counters.p;
        P.survivors_total = S.counters.p + 1;
        P.mask_fold = D->params.mask_fold;
        P.mask_single = D->params.mask_single;
        // reject iff F_D > 2k (ceil_half(F_D) > k, dictionary.hpp:102-106); the
        // one-hot count form counts every differing field twice
        P.thr = o.use_filter ? (onehot ? 4 * o.k : 2 * o.k) : 1 << 20;
        P.k = o.k;
        P.fold = D->params.variant == FPG_COUNT ? D->params.b
               : D->params.variant == FPG_POSITION ? D->params.p : 1;
        P.q_matches = S.qsurv.p + nq;
        P.match_total = S.counters.p + 5;
    }
    // K2, then K4 speculatively on the segmented path (no host round trip);
    // the one sync reads the counters and redoes what they rule out: a
    // larger output buffer (rescan), or sorts the queries with > kSegMax
    // matches (k_seg_sort_big).
    S.offsets.reserve(nq + 1);
    S.big_list.reserve(nq);
    const bool warp_sort = nq != 0;
    // Candidate buffer of the bit-sliced path: records per K2 + K3 round.
    // FPG_CAND_MAX_MB bounds it (default 48 GB, and a third of the free
    // device memory); FPG_CAND_MAX (records) is the tests' override.
    auto cand_limit = [&]() -> uint64_t {
        size_t free_b = 0, total_b = 0;
        CK(cudaMemGetInfo(&free_b, &total_b));
        const double mb = env_double("FPG_CAND_MAX_MB", 49152.0);
        uint64_t rec = (uint64_t)std::min<double>(mb * 1048576.0, (double)(free_b + S.cand.cap * sizeof(uint4)) / 3.0) /
                       sizeof(uint4);
        const double forced = env_double("FPG_CAND_MAX", 0.0);
        if (forced > 0) rec = (uint64_t)forced;
        if (S.cand_fail) rec = std::min<uint64_t>(rec, S.cand_fail / 2);  // an allocation of cand_fail records was refused
        return std::max<uint64_t>(rec, 1024);
    };
    if (use_slice && !S.cand_cap) {
        S.cand_cap = std::min<uint64_t>(std::max<uint64_t>(executed / 256, 1u << 20), cand_limit());
        S.cand_rounds = 1;
    }
    for (bool first = true;; first = false) {
        S.out.reserve(S.out_cap);
        S.ids.reserve(S.out.cap);
        P.out = VP.out = S.out.p;
        P.out_cap = VP.out_cap = S.out.cap;
        if (!first) {  // rescan after growing a buffer (K1 zeroed them the first time)
            CK(cudaMemsetAsync(S.counters.p, 0, kNumCounters * sizeof(unsigned long long), st));
            if (nq) CK(cudaMemsetAsync(S.qsurv.p, 0, 2 * nq * sizeof(uint32_t), st));
        }
        CK(cudaEventRecord(S.ev[1], st));
        if (use_slice) {
            // a refused allocation (fragmented or shared device memory) halves the
            // buffer; the run then takes more rounds instead of failing
            while (S.cand.cap < S.cand_cap) {
                try {
                    S.cand.reserve(S.cand_cap);
                } catch (const Error&) {
                    cudaGetLastError();
                    if (S.cand_cap <= (1u << 20)) throw;
                    S.cand_fail = S.cand_cap;  // bounds the later limits (cand_limit)
                    S.cand_cap = std::max<uint64_t>(S.cand_cap / 2, 1u << 20);
                }
            }
            SP.cand = S.cand.p;
            SP.cand_cap = S.cand_cap;
            const uint32_t R = S.cand_rounds;
            while (S.ev_k3.size() < 2 * (size_t)R) {
                cudaEvent_t e = nullptr;
                CK(cudaEventCreate(&e));
                S.ev_k3.push_back(e);
            }
            // round r scans every R-th tile of each plan from tile r on: the plan's
            // mix of lengths (and so of candidates per tile) in every round
            auto share = [&](const std::vector<fpg::SliceTile>& pl, uint32_t r) -> uint32_t {
                return pl.size() > r ? (uint32_t)((pl.size() - r + R - 1) / R) : 0u;
            };
            SP.tile_stride = R;
            // barrier-free tiles for plans whose tiles were shrunk (small batches)
            SP.no_barrier = S.plan_small ? 1 : 0;
            {
                const double nb_env = env_double("FPG_NO_BARRIER", -1.0);  // A/B and tests: 0 / 1 forces it
                if (nb_env >= 0) SP.no_barrier = nb_env != 0.0;
            }
            for (uint32_t r = 0; r < R; ++r) {
                if (r) {  // the rounds reuse the tile counters and the record buffer
                    CK(cudaMemsetAsync(S.counters.p + 2, 0, sizeof(unsigned long long), st));
                    CK(cudaMemsetAsync(S.counters.p + 9, 0, sizeof(unsigned long long), st));
                    CK(cudaMemsetAsync(S.counters.p + 11, 0, sizeof(unsigned long long), st));
                    CK(cudaMemsetAsync(S.counters.p + 14, 0, sizeof(unsigned long long), st));
                }
                SP.tile_off = r;
                const uint32_t na = share(splan, r), nx = share(splan_x, r);
                if (na) {
                    dispatch_slice(D->scheme, D->params.nsig, S.stiles.p, na, SP, st, sh.device);
                    ++S.launches;
                }
                if (nx) {
                    // the exact path: position-code planes instead of sig', own tile
                    // counter and pair count
                    fpg::SliceParams SX = SP;
                    SX.planes = W.xplanes.p;
                    SX.q_sigp = Q.xc.p;
                    SX.tile_counter = reinterpret_cast<unsigned int*>(S.counters.p + 9);
                    SX.scanned = S.counters.p + 10;
                    fpg_host::dispatch_slice_16x(field_width_of(D->scheme), S.stiles_x.p, nx, SX, st, sh.device);
                    ++S.launches;
                }
                // K3 right behind: the record count stays on the device
                CK(cudaEventRecord(S.ev_k3[2 * r], st));
                if (na || nx) {
                    // strings of up to 16 bytes compare from four registers each, else eight
                    // (Hamming only compares equal lengths)
                    const bool short16 = W.max_len <= 16 && (o.metric == FPG_HAMMING || Q.max_len <= 16);
                    auto kv = short16 ? fpg::k_verify<4> : fpg::k_verify<8>;
                    // one resident wave: the warps in flight then work on one window of
                    // the record stream (records of one K2 moment share a slab range), and
                    // the buffer is swept once (FPG_VERIFY_CTAS overrides, A/B runs)
                    static int resident[2][64] = {{0}};
                    const int dv = sh.device & 63;
                    if (!resident[short16][dv]) {
                        int sms = 148, per_sm = 0;
                        CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, sh.device));
                        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kv, fpg::kVerifyThreads, 0));
                        resident[short16][dv] = sms * std::max(per_sm, 1);
                    }
                    static const unsigned forced = (unsigned)env_double("FPG_VERIFY_CTAS", 0.0);
                    const unsigned vgrid = forced ? forced : (unsigned)resident[short16][dv];
                    kv<<<vgrid, fpg::kVerifyThreads, 0, st>>>(VP, S.cand.p, S.counters.p + 11, S.cand_cap, S.counters.p + 5,
                                                              S.counters.p + 3, S.counters.p + 12, S.counters.p + 13,
                                                              S.counters.p + 14);
                    CK(cudaGetLastError());
                    ++S.launches;
                }
                CK(cudaEventRecord(S.ev_k3[2 * r + 1], st));
            }
        } else if (!plan.empty()) {
            dispatch_scan(D->params, D->params.onehot && !from_slice, o.want_stats != 0, S.tiles.p,
                          (uint32_t)plan.size(), P, st, sh.device);
            ++S.launches;
        }
        CK(cudaEventRecord(S.ev[2], st));
        if (ext_stats && nq) {
            // per-query fingerprint survivors from the histograms (k = 0: the
            // query's own fingerprint only, the first mask)
            const int span = o.metric == FPG_HAMMING ? 0 : o.k;
            const int all_len = (o.metric == FPG_LEVENSHTEIN && !o.length_prefilter) ? 1 : 0;
            fpg::k_fp_stats<<<(unsigned)std::min<uint64_t>(cdiv(nq, 8), 148 * 16), 256, 0, st>>>(
                Q.fp.p, Q.len_b.p, Q.ids.p, nq, W.fph.p, W.d_hslot.p, W.nh, W.max_len, W.d_hdelta.p,
                o.k == 0 ? 1 : W.n_hdelta, span, all_len, S.qsurv.p, S.counters.p + 1);
            CK(cudaGetLastError());
            ++S.launches;
        }
        // K4: offsets = exclusive scan of the per-query match counts, keys
        // scattered into their query's segment, then each segment of <=
        // kSegMax matches sorted by one warp; larger ones are listed.
        if (nq) {  // accumulated in 64 bits: a batch may hold >= 2^32 matches
            size_t tmp = 0;
            CK(cub::DeviceScan::ExclusiveScan(nullptr, tmp, S.qsurv.p + nq, S.offsets.p, cuda::std::plus<>{}, uint64_t(0),
                                              (int)nq, st));
            S.cub_tmp.reserve(tmp);
            CK(cub::DeviceScan::ExclusiveScan(S.cub_tmp.p, tmp, S.qsurv.p + nq, S.offsets.p, cuda::std::plus<>{}, uint64_t(0),
                                              (int)nq, st));
        }
        fpg::k_seg_scatter<<<kScatterBlocks, 256, 0, st>>>(S.out.p, S.counters.p, S.counters.p + 5, S.out.cap,
                                                           S.offsets.p, S.qsurv.p + nq, S.ids.p, S.offsets.p + nq,
                                                           W.ids.p, D->id_base + sh.base);
        CK(cudaGetLastError());
        S.launches += 2;
        if (warp_sort) {
            fpg::k_seg_sort<<<(unsigned)cdiv(nq * 32, 256), 256, 0, st>>>(S.offsets.p, nq, S.out.cap, S.ids.p,
                                                                           S.counters.p + 4, S.big_list.p,
                                                                           S.counters.p + 7);
            CK(cudaGetLastError());
            ++S.launches;
        }
        CK(cudaMemcpyAsync(S.h_counters.p, S.counters.p, kNumCounters * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        bool redo = false;
        if (use_slice && S.h_counters.p[12]) {
            // a round's candidate records did not fit: a larger buffer up to the
            // limit, then more rounds (capacity x rounds grows by >= 1.25 per attempt)
            const double need = 1.25 * (double)S.h_counters.p[13] * S.cand_rounds;
            const uint64_t lim = cand_limit();
            S.cand_cap = (uint64_t)std::min<double>((double)lim, need);
            S.cand_rounds = (uint32_t)std::max<double>(1.0, std::ceil(need / (double)S.cand_cap));
            if (S.cand_rounds > splan.size() + splan_x.size())
                throw Error(FPG_ENOMEM, "candidate buffer too small for one K2 tile (FPG_CAND_MAX_MB)");
            redo = true;
        }
        if (S.h_counters.p[0] > S.out.cap) {  // reserved key slots did not fit
            S.out_cap = S.h_counters.p[0] + S.h_counters.p[0] / 4 + 1024;
            redo = true;
        }
        if (!redo) break;  // else grow and rescan
    }
    S.cand_records = use_slice ? S.h_counters.p[13] : 0;
    S.total = S.h_counters.p[5];
    S.survivors = S.h_counters.p[1];
    S.candidates = S.h_counters.p[3];
    S.scanned = use_slice ? S.h_counters.p[6] + S.h_counters.p[10] : executed;
    S.scanned_x = use_slice ? S.h_counters.p[10] : 0;

    S.ids_out = S.ids.p;
    bool cub_sort = false;
    if (S.total && S.h_counters.p[4]) {
        // queries with more than kSegMax matches: one CTA each sorts them in
        // place (ids2 is its bucket scratch)
        S.ids2.reserve(S.total);
        const uint64_t nbig = S.h_counters.p[7];
        fpg::k_seg_sort_big<<<(unsigned)std::min<uint64_t>(nbig, 148 * 8), fpg::kBigThreads, 0, st>>>(
            S.offsets.p, S.big_list.p, nbig, S.ids.p, S.ids2.p, S.counters.p + 8);
        CK(cudaGetLastError());
        ++S.launches;
        CK(cudaMemcpyAsync(S.h_counters.p + 8, S.counters.p + 8, sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        cub_sort = S.h_counters.p[8] != 0;  // a bucket too large (very skewed ids): sort everything with CUB
    }
    if (S.total && cub_sort) {
        if (S.total >= (1ull << 31)) throw Error(FPG_EINVAL, "more than 2^31 - 1 matches in one shard's batch");
        S.ids2.reserve(S.total);
        size_t tmp = 0;
        CK(cub::DeviceSegmentedSort::SortKeys(nullptr, tmp, S.ids.p, S.ids2.p, (int)S.total, (int)nq, S.offsets.p,
                                              S.offsets.p + 1, st));
        S.cub_tmp.reserve(tmp);
        CK(cub::DeviceSegmentedSort::SortKeys(S.cub_tmp.p, tmp, S.ids.p, S.ids2.p, (int)S.total, (int)nq,
                                              S.offsets.p, S.offsets.p + 1, st));
        S.ids_out = S.ids2.p;
        ++S.launches;
    }
    CK(cudaEventRecord(S.ev[3], st));
    CK(cudaEventSynchronize(S.ev[3]));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, S.ev[0], S.ev[3]));
    S.run_ms = ms;
    CK(cudaEventElapsedTime(&ms, S.ev[1], S.ev[2]));
    S.filter_ms = ms;
    S.verify_ms = 0;
    if (use_slice) {  // K2 time = the rounds' time minus their K3 launches
        for (uint32_t r = 0; r < S.cand_rounds; ++r) {
            CK(cudaEventElapsedTime(&ms, S.ev_k3[2 * r], S.ev_k3[2 * r + 1]));
            S.verify_ms += ms;
        }
        S.filter_ms -= S.verify_ms;
    }
    g_launches += S.launches;
}

void download_shard(fpg_batch* B, ShardBatch& S, bool stats) {
    CK(cudaSetDevice(S.sh->device));
    cudaStream_t st = S.stream;
    const uint64_t nq = B->nq;
    S.h_offsets.reserve(nq + 1);
    S.h_ids.reserve(S.total);
    CK(cudaMemcpyAsync(S.h_offsets.p, S.offsets.p, (nq + 1) * sizeof(uint64_t), cudaMemcpyDeviceToHost, st));
    if (S.total) CK(cudaMemcpyAsync(S.h_ids.p, S.ids_out, S.total * sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
    if (stats && nq) {
        S.h_qsurv.reserve(nq);
        CK(cudaMemcpyAsync(S.h_qsurv.p, S.qsurv.p, nq * sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
    }
    CK(cudaStreamSynchronize(st));
}

void check_opts(const fpg_dict* D, const fpg_query_options* o) {
    if (!o) throw Error(FPG_EINVAL, "null options");
    if (o->metric != FPG_HAMMING && o->metric != FPG_LEVENSHTEIN) throw Error(FPG_EINVAL, "unknown metric");
    if (o->use_filter && !supports(D->scheme.variant, o->metric))
        throw Error(FPG_EINVAL, "scheme does not filter for this metric");
    if (o->k < 0) throw Error(FPG_EINVAL, "k must be >= 0");
    if (o->k > fpg::kMaxK)
        throw Error(FPG_EUNSUPPORTED, "GPU scan supports k <= " + std::to_string(fpg::kMaxK) + ", got " +
                                          std::to_string(o->k));
}

// sync = false (fpg_query_batch): the caller's buffers stay valid until the
// call returns, so the copies may still be in flight when upload returns.
void upload(fpg_batch* B, const uint8_t* qbytes, const uint64_t* qoffsets, uint64_t nq, bool sync = true) {
    const auto t0 = std::chrono::steady_clock::now();
    if (nq && !qoffsets) throw Error(FPG_EINVAL, "null query offsets");
    if (nq >= (1ull << 31)) throw Error(FPG_EINVAL, "too many queries in one batch");
    B->nq = nq;
    B->qlen.resize(nq);
    const int L1 = fpg::kMaxLen + 1;
    B->qcount.assign(L1, 0);
    const uint64_t q0 = nq ? qoffsets[0] : 0;
    // Lengths, their histogram and (below) the stable counting sort run on up
    // to 16 host threads over contiguous chunks of a large batch: chunk c
    // scatters its queries behind those of the chunks before it.
    const unsigned hw = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
    const uint64_t C = std::max<uint64_t>(1, std::min<uint64_t>(hw, nq >> 16));
    auto chunk_lo = [&](uint64_t c) { return nq * c / C; };
    auto chunks = [&](auto&& f) {
        if (C == 1) {
            f(uint64_t(0));
            return;
        }
        std::vector<std::thread> th;
        for (uint64_t c = 0; c < C; ++c) th.emplace_back([&f, c] { f(c); });
        for (auto& x : th) x.join();
    };
    std::vector<uint64_t> cmax(C, 0);
    std::vector<std::vector<uint32_t>> chist(C);
    chunks([&](uint64_t c) {
        std::vector<uint32_t>& h = chist[c];
        h.assign(L1, 0);
        uint64_t mx = 0;
        for (uint64_t i = chunk_lo(c); i < chunk_lo(c + 1); ++i) {
            const uint64_t len = qoffsets[i + 1] - qoffsets[i];  // wraps (huge) if not ascending
            mx = len > mx ? len : mx;
            B->qlen[i] = (uint32_t)len;
            if (len < (uint64_t)L1) ++h[len];
        }
        cmax[c] = mx;
    });
    uint64_t len_max = 0;
    for (uint64_t c = 0; c < C; ++c) len_max = std::max(len_max, cmax[c]);
    if (len_max > (uint64_t)fpg::kMaxLen) {
        for (uint64_t i = 0; i < nq; ++i)
            if (qoffsets[i + 1] < qoffsets[i]) throw Error(FPG_EINVAL, "query offsets not ascending");
        throw Error(FPG_EINVAL, "query longer than FPG_MAX_WORD_LEN");
    }
    for (uint64_t c = 0; c < C; ++c)
        for (uint64_t L = 0; L <= len_max; ++L) B->qcount[L] += chist[c][L];
    if (nq && qoffsets[nq] > q0 && !qbytes) throw Error(FPG_EINVAL, "null query bytes");
    // Length buckets: stable counting sort of the query ids (the layout K1
    // writes, with the padded-byte offset of every bucket).
    B->qstart.assign(L1, 0);
    B->qbbase.assign(L1, 0);
    B->h_start.reserve(L1);
    B->h_bbase.reserve(L1);
    B->h_order.reserve(nq);
    uint64_t pos = 0, bpos = 0;
    B->qmax_len = 0;
    for (int L = 0; L <= (int)len_max; ++L) {
        B->qstart[L] = (uint32_t)pos;
        B->qbbase[L] = bpos;
        B->h_start.p[L] = (uint32_t)pos;
        B->h_bbase.p[L] = bpos;
        pos += B->qcount[L];
        bpos += (uint64_t)B->qcount[L] * stride_of(L);
        if (B->qcount[L]) B->qmax_len = L;
    }
    // lengths above the longest query: empty buckets at the end
    std::fill(B->qstart.begin() + len_max + 1, B->qstart.end(), (uint32_t)pos);
    std::fill(B->qbbase.begin() + len_max + 1, B->qbbase.end(), bpos);
    std::fill(B->h_start.p + len_max + 1, B->h_start.p + L1, (uint32_t)pos);
    std::fill(B->h_bbase.p + len_max + 1, B->h_bbase.p + L1, bpos);
    B->qtotal_bytes = bpos;
    {
        // chunk c's first slot per length: the bucket start plus the earlier chunks' counts
        std::vector<uint32_t> run(B->qstart.begin(), B->qstart.begin() + len_max + 1);
        for (uint64_t c = 0; c < C; ++c)
            for (uint64_t L = 0; L <= len_max; ++L) {
                const uint32_t n_cl = chist[c][L];
                chist[c][L] = run[L];
                run[L] += n_cl;
            }
        chunks([&](uint64_t c) {
            std::vector<uint32_t>& cur = chist[c];
            for (uint64_t i = chunk_lo(c); i < chunk_lo(c + 1); ++i) B->h_order.p[cur[B->qlen[i]]++] = (uint32_t)i;
        });
    }
    const uint64_t nbytes = nq ? qoffsets[nq] - q0 : 0;
    const auto t1 = std::chrono::steady_clock::now();
    for_each_shard(B->sb.size(), [&](size_t i) {
        ShardBatch& S = *B->sb[i];
        CK(cudaSetDevice(S.sh->device));
        cudaStream_t st = S.stream;
        S.qblob.reserve(nbytes + 16);
        S.qoffs.reserve(nq + 1);
        S.qorder.reserve(nq);
        // the tile plan and the bucket tables depend on the batch only
        // through its length histogram
        const bool new_hist = S.plan_qcount != B->qcount;
        if (new_hist) {
            S.plan_valid = false;
            S.plan_qcount = B->qcount;
        }
        Collection& Q = S.queries;
        Q.n = nq;
        Q.count = B->qcount;
        Q.start = B->qstart;
        Q.byte_base = B->qbbase;
        Q.max_len = B->qmax_len;
        Q.total_bytes = B->qtotal_bytes;
        Q.d_start.reserve(L1);
        Q.d_byte_base.reserve(L1);
        if (nbytes) CK(cudaMemcpyAsync(S.qblob.p, qbytes + q0, nbytes, cudaMemcpyHostToDevice, st));
        if (nq) {
            CK(cudaMemcpyAsync(S.qorder.p, B->h_order.p, nq * sizeof(uint32_t), cudaMemcpyHostToDevice, st));
            if (q0 == 0) {
                CK(cudaMemcpyAsync(S.qoffs.p, qoffsets, (nq + 1) * sizeof(uint64_t), cudaMemcpyHostToDevice, st));
            } else {
                std::vector<uint64_t> rebased(nq + 1);
                for (uint64_t j = 0; j <= nq; ++j) rebased[j] = qoffsets[j] - q0;
                CK(cudaMemcpyAsync(S.qoffs.p, rebased.data(), (nq + 1) * sizeof(uint64_t), cudaMemcpyHostToDevice, st));
            }
        }
        if (new_hist) {
            CK(cudaMemcpyAsync(Q.d_start.p, B->h_start.p, L1 * sizeof(uint32_t), cudaMemcpyHostToDevice, st));
            CK(cudaMemcpyAsync(Q.d_byte_base.p, B->h_bbase.p, L1 * sizeof(uint64_t), cudaMemcpyHostToDevice, st));
        }
        if (sync) CK(cudaStreamSynchronize(st));  // caller buffers may be reused once upload returns
    });
    B->uploaded = true;
    B->upload_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    if (g_trace) {
        const auto t2 = std::chrono::steady_clock::now();
        std::fprintf(stderr, "fpg upload: host bucketing %.1f us, h2d %.1f us\n",
                     std::chrono::duration<double, std::micro>(t1 - t0).count(),
                     std::chrono::duration<double, std::micro>(t2 - t1).count());
    }
}

void run(fpg_batch* B, const fpg_query_options* o) {
    check_opts(B->dict, o);
    if (!B->uploaded) throw Error(FPG_EINVAL, "fpg_batch_run before fpg_batch_upload");
    B->ran = false;  // stays false if a shard fails: download refuses stale results
    B->opt = *o;
    for_each_shard(B->sb.size(), [&](size_t i) { run_shard(B->dict, B, *B->sb[i], *o); });
    B->ran = true;
}

// Assembles the caller-visible CSR (+ QueryStats) from the shards.
void download(fpg_batch* B, fpg_result* out) {
    if (!B->ran) throw Error(FPG_EINVAL, "fpg_batch_download before fpg_batch_run");
    const fpg_query_options& o = B->opt;
    const bool stats = o.want_stats != 0;
    const auto t0 = std::chrono::steady_clock::now();
    const uint64_t nq = B->nq;
    std::memset(out, 0, sizeof(*out));
    out->nq = nq;
    uint64_t total = 0;
    for (auto& s : B->sb) total += s->total;
    out->total = total;
    PinnedPool& pool = pinned_pool();
    out->offsets = static_cast<uint64_t*>(pool.get(sizeof(uint64_t) * (nq + 1)));
    out->word_ids = static_cast<uint32_t*>(pool.get(sizeof(uint32_t) * std::max<uint64_t>(total, 1)));
    if (B->sb.size() == 1) {
        // one shard: the CSR goes straight into the result's pinned arrays
        ShardBatch& S = *B->sb[0];
        CK(cudaSetDevice(S.sh->device));
        cudaStream_t st = S.stream;
        CK(cudaMemcpyAsync(out->offsets, S.offsets.p, (nq + 1) * sizeof(uint64_t), cudaMemcpyDeviceToHost, st));
        if (total) CK(cudaMemcpyAsync(out->word_ids, S.ids_out, total * sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
        if (stats && nq) {
            S.h_qsurv.reserve(nq);
            CK(cudaMemcpyAsync(S.h_qsurv.p, S.qsurv.p, nq * sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
        }
        CK(cudaStreamSynchronize(st));
    } else {
        for_each_shard(B->sb.size(), [&](size_t i) { download_shard(B, *B->sb[i], stats); });
    }
    const auto t1 = std::chrono::steady_clock::now();
    B->download_ms = std::chrono::duration<double, std::milli>(t1 - t0).count();
    if (B->sb.size() > 1) {
        // Shards own ascending contiguous id ranges: concatenating each query's
        // shard rows in shard order yields ascending ids (oracle order).
        uint64_t pos = 0;
        for (uint64_t q = 0; q < nq; ++q) {
            out->offsets[q] = pos;
            for (auto& s : B->sb) pos += s->h_offsets.p[q + 1] - s->h_offsets.p[q];
        }
        out->offsets[nq] = pos;
        parallel_ranges(nq, 1u << 14, [&](uint64_t qlo, uint64_t qhi) {
            for (uint64_t q = qlo; q < qhi; ++q) {
                uint64_t at = out->offsets[q];
                for (auto& s : B->sb) {
                    const uint64_t a = s->h_offsets.p[q], b = s->h_offsets.p[q + 1];
                    if (b > a) std::memcpy(out->word_ids + at, s->h_ids.p + a, sizeof(uint32_t) * (b - a));
                    at += b - a;
                }
            }
        });
    }
    if (stats) {
        out->stats = static_cast<uint64_t*>(pool.get(FPG_NSTATS * sizeof(uint64_t) * std::max<uint64_t>(nq, 1)));
        const fpg_dict* D = B->dict;
        const uint64_t N = D->n;
        // length-compatible words per query length (QueryStats bookkeeping,
        // dictionary.hpp:89-101): N for Levenshtein without the prefilter
        const int L1 = fpg::kMaxLen + 1;
        const bool all = o.metric == FPG_LEVENSHTEIN && !o.length_prefilter;
        std::vector<uint64_t> comp_of(B->qmax_len + 1, N);
        if (!all)
            for (int lq = 0; lq <= B->qmax_len; ++lq) {
                const int lo = o.metric == FPG_HAMMING ? lq : std::max(0, lq - o.k);
                const int hi = o.metric == FPG_HAMMING ? lq : std::min(L1 - 1, lq + o.k);
                uint64_t c = 0;
                for (int L = lo; L <= hi; ++L) c += D->len_count[L];
                comp_of[lq] = c;
            }
        const size_t G = B->sb.size();
        parallel_ranges(nq, 1u << 16, [&](uint64_t qlo, uint64_t qhi) {
            for (uint64_t q = qlo; q < qhi; ++q) {
                uint64_t surv = 0;
                for (size_t g = 0; g < G; ++g) surv += B->sb[g]->h_qsurv.p[q];
                const uint64_t comp = comp_of[B->qlen[q]];
                uint64_t* st = out->stats + FPG_NSTATS * q;
                const uint64_t verified = o.use_filter ? surv : comp;
                st[FPG_STAT_COMPARED] = N;
                st[FPG_STAT_REJECTED_BY_LENGTH] = N - comp;
                st[FPG_STAT_REJECTED_BY_FINGERPRINT] = comp - verified;
                st[FPG_STAT_VERIFIED] = verified;
                st[FPG_STAT_MATCHES] = out->offsets[q + 1] - out->offsets[q];
            }
        });
    }
    B->assemble_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t1).count();
    if (g_trace) {
        const auto t2 = std::chrono::steady_clock::now();
        std::fprintf(stderr, "fpg download: d2h %.1f us, assemble %.1f us\n",
                     std::chrono::duration<double, std::micro>(t1 - t0).count(),
                     std::chrono::duration<double, std::micro>(t2 - t1).count());
    }
}

// Chooses the K2 path and the sig' map: non-letter bytes of the dictionary,
// ranked by frequency (descending, then byte), dealt round robin onto S
// one-bit fields (S = 0 / 8 / 10 / 12 / 16 by how many such bytes exist; FPG_SIGP_BITS
// overrides).  FPG_SLICE=0 selects the generic k_scan for A/B runs.
void configure_slice(fpg_dict& D, const std::vector<unsigned long long>& hist) {
    const char* e = std::getenv("FPG_SLICE");
    D.slice = slice_supported(D.scheme) && !(e && e[0] == '0');
    std::vector<int> others;
    for (int c = 0; c < 256; ++c)
        if (hist[c] && D.params.slot[c] < 0) others.push_back(c);
    std::stable_sort(others.begin(), others.end(), [&](int a, int b) { return hist[a] > hist[b]; });
    auto snap = [](size_t v) { return v == 0 ? 0 : v <= 8 ? 8 : v <= 10 ? 10 : v <= 12 ? 12 : 16; };
    // W = 32 takes at most 12 sig' fields: NPT = 44 leaves one slab per lane,
    // yet every W = 32 cell of configs 3 and 5 ran 4-10% faster than with 8
    // (fewer candidates).  No sig' when it cannot pay (measured): <= 4 other
    // symbols, or a 64-bit count fingerprint (16 four-bit fields already
    // leave few candidates).
    int S = snap(std::min<size_t>(others.size(), D.scheme.width == 32 ? 12 : 16));
    if (others.size() <= 4 || (D.scheme.width == 64 && D.scheme.variant == FPG_COUNT)) S = 0;
    if (const char* sb = std::getenv("FPG_SIGP_BITS")) S = snap((size_t)std::max(0, std::atoi(sb)));
    std::memset(D.params.sigbit, -1, sizeof(D.params.sigbit));
    if (S)
        for (size_t r = 0; r < others.size(); ++r) D.params.sigbit[others[r]] = (int8_t)(r % S);
    D.params.nsig = S;
    D.npt = D.scheme.width + S;
    // exact Hamming path of short words (K2 X, fpg_slice.cuh): W = 16 and at
    // most 31 distinct dictionary bytes, coded densely in kXBits bits; bytes
    // the dictionary lacks share code 31, which no dictionary word uses
    int distinct = 0;
    for (int c = 0; c < 256; ++c) distinct += hist[c] ? 1 : 0;
    std::memset(D.params.xcode, (1 << fpg::kXBits) - 1, sizeof(D.params.xcode));
    D.params.xlen = 0;
    if (D.slice && D.scheme.width == 16 && distinct < (1 << fpg::kXBits)) {
        int r = 0;
        for (int c = 0; c < 256; ++c)
            if (hist[c]) D.params.xcode[c] = (uint8_t)r++;
        D.params.xlen = fpg::kXLen;
    }
}

void make_batch(fpg_dict* D, fpg_batch** out) {
    auto B = std::make_unique<fpg_batch>();
    B->dict = D;
    for (auto& sh : D->shards) {
        auto S = std::make_unique<ShardBatch>();
        S->sh = sh.get();
        CK(cudaSetDevice(sh->device));
        CK(cudaStreamCreateWithFlags(&S->stream, cudaStreamNonBlocking));
        B->sb.push_back(std::move(S));
    }
    *out = B.release();
}

}  // namespace

extern "C" {

const char* fpg_last_error(void) { return g_last_error.c_str(); }
int fpg_abi_version(void) { return FPG_ABI_VERSION; }

int fpg_device_count(int* count) {
    return guarded([&] {
        int n = 0;
        CK(cudaGetDeviceCount(&n));
        *count = n;
    });
}

int fpg_letter_capacity(int32_t variant, int32_t width, int32_t b, int32_t p) {
    const int c = capacity(variant, width, b, p);
    if (c < 0) g_last_error = "invalid scheme parameters";
    return c;
}

int fpg_scheme_validate(const fpg_scheme* scheme) {
    return guarded([&] { validate(scheme); });
}

int fpg_scheme_supports(const fpg_scheme* scheme, int32_t metric) {
    return scheme && supports(scheme->variant, metric) ? 1 : 0;
}

namespace {

std::vector<int32_t> checked_devices(const int32_t* devices, int32_t ndevices) {
    std::vector<int32_t> devs;
    if (devices && ndevices > 0) devs.assign(devices, devices + ndevices);
    else devs.push_back(0);
    int ndev = 0;
    CK(cudaGetDeviceCount(&ndev));
    for (int d : devs)
        if (d < 0 || d >= ndev) throw Error(FPG_EINVAL, "device " + std::to_string(d) + " not present");
    return devs;
}

std::unique_ptr<fpg_dict> new_dict(const fpg_scheme* scheme, uint64_t id_base, const std::vector<int32_t>& devs) {
    auto D = std::make_unique<fpg_dict>();
    D->scheme = *scheme;
    D->params = make_params(*scheme);
    D->id_base = id_base;
    D->len_count.assign(fpg::kMaxLen + 1, 0);
    for (int32_t d : devs) {
        auto sh = std::make_unique<Shard>();
        sh->device = d;
        D->shards.push_back(std::move(sh));
    }
    return D;
}

// Contiguous input-order id ranges, one per shard.
void assign_ranges(fpg_dict& D, uint64_t n) {
    if (n >= (1ull << 32) - 1) throw Error(FPG_EINVAL, "dictionary too large for 32-bit ids");
    if (D.id_base + n > (1ull << 32)) throw Error(FPG_EINVAL, "id_base + n exceeds 32-bit ids");
    D.n = n;
    const size_t G = D.shards.size();
    for (size_t g = 0; g < G; ++g) {
        D.shards[g]->base = n * g / G;
        D.shards[g]->n = n * (g + 1) / G - D.shards[g]->base;
        // the shard's CUB sorts index with int
        if (D.shards[g]->n >= (1ull << 31)) throw Error(FPG_EINVAL, "more than 2^31 - 1 words in one shard");
    }
}

void byte_histogram(const uint8_t* d_bytes, uint64_t nbytes, unsigned long long* d_hist, cudaStream_t st) {
    CK(cudaMemsetAsync(d_hist, 0, 256 * sizeof(unsigned long long), st));
    if (nbytes) {
        fpg::k_hist256<<<(unsigned)std::min<uint64_t>(cdiv(nbytes, 256), 4096), 256, 0, st>>>(d_bytes, nbytes, d_hist);
        CK(cudaGetLastError());
    }
}

// Phase 2 of construction, after every shard's strings are on its device
// (sh.blob, sh.offs + offs_at[g]) and `hist` counts the dictionary's bytes:
// the K2 path and sig' map, then fingerprints, length buckets, padded bytes
// and planes per shard.
void finish_dict(fpg_dict& D, const std::vector<unsigned long long>& hist, const std::vector<uint64_t>& offs_at,
                 std::chrono::steady_clock::time_point t0) {
    configure_slice(D, hist);
    for_each_shard(D.shards.size(), [&](size_t g) {
        Shard& sh = *D.shards[g];
        CK(cudaSetDevice(sh.device));
        sh.dict.build(sh.blob.p, sh.offs.p + offs_at[g], sh.n, D.params, sh.stream,
                      D.slice ? kSliceDict : kGenericDict, D.npt);
        CK(cudaStreamSynchronize(sh.stream));
        sh.dict.stage_finish();
        sh.dict.drop_scratch();
        sh.blob.release();
        sh.offs.release();
    });
    for (auto& sh : D.shards)
        for (int L = 0; L <= fpg::kMaxLen; ++L) D.len_count[L] += sh->dict.count[L];
    D.build_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

struct IsNewline {
    const uint8_t* t;
    __device__ bool operator()(uint64_t i) const { return t[i] == '\n'; }
};
struct NotNewline {
    __device__ bool operator()(uint8_t c) const { return c != '\n'; }
};

// Word i of a newline-separated text, after the newlines are removed
// (read_word_lines, corpus.hpp:116-125: a trailing newline ends the last word,
// empty lines are empty words): offsets[i] = nl[i-1] + 1 - i, offsets[n] =
// bytes left.
__global__ void k_text_offsets(const uint64_t* __restrict__ nl, uint64_t n, uint64_t kept,
                               uint64_t* __restrict__ offsets) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i > n) return;
    offsets[i] = i == 0 ? 0 : i == n ? kept : nl[i - 1] + 1 - i;
}

}  // namespace

int fpg_dict_create(const uint8_t* bytes, const uint64_t* offsets, uint64_t n, const fpg_scheme* scheme,
                    const int32_t* devices, int32_t ndevices, uint64_t id_base, fpg_dict** out) {
    return guarded([&] {
        validate(scheme);
        if (!out) throw Error(FPG_EINVAL, "null output handle");
        if (n && !offsets) throw Error(FPG_EINVAL, "null dictionary offsets");
        if (n && offsets[n] > offsets[0] && !bytes) throw Error(FPG_EINVAL, "null dictionary bytes");
        const std::vector<int32_t> devs = checked_devices(devices, ndevices);
        auto t0 = std::chrono::steady_clock::now();
        auto D = new_dict(scheme, id_base, devs);
        assign_ranges(*D, n);
        const size_t G = devs.size();
        // Phase 1: upload each shard's strings and count its bytes (sig' ranking).
        for_each_shard(G, [&](size_t g) {
            Shard& sh = *D->shards[g];
            CK(cudaSetDevice(sh.device));
            CK(cudaStreamCreateWithFlags(&sh.stream, cudaStreamNonBlocking));
            const uint64_t b0 = sh.n ? offsets[sh.base] : 0;
            const uint64_t nbytes = sh.n ? offsets[sh.base + sh.n] - b0 : 0;
            sh.blob.reserve(nbytes + 16);  // K1 reads whole aligned words past the end
            sh.offs.reserve(sh.n + 1);
            std::vector<uint64_t> local(sh.n + 1);
            for (uint64_t i = 0; i <= sh.n; ++i) local[i] = (sh.n ? offsets[sh.base + i] : 0) - b0;
            if (nbytes) CK(cudaMemcpyAsync(sh.blob.p, bytes + b0, nbytes, cudaMemcpyHostToDevice, sh.stream));
            CK(cudaMemcpyAsync(sh.offs.p, local.data(), (sh.n + 1) * sizeof(uint64_t), cudaMemcpyHostToDevice, sh.stream));
            sh.d_hist.reserve(256);
            sh.h_hist.reserve(256);
            byte_histogram(sh.blob.p, nbytes, sh.d_hist.p, sh.stream);
            CK(cudaMemcpyAsync(sh.h_hist.p, sh.d_hist.p, 256 * sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                               sh.stream));
            CK(cudaStreamSynchronize(sh.stream));
        });
        std::vector<unsigned long long> hist(256, 0);
        for (auto& sh : D->shards)
            for (int c = 0; c < 256; ++c) hist[c] += sh->h_hist.p[c];
        finish_dict(*D, hist, std::vector<uint64_t>(G, 0), t0);
        *out = D.release();
    });
}

int fpg_dict_create_from_text(const uint8_t* text, uint64_t nbytes, const fpg_scheme* scheme,
                              const int32_t* devices, int32_t ndevices, uint64_t id_base, fpg_dict** out) {
    return guarded([&] {
        validate(scheme);
        if (!out) throw Error(FPG_EINVAL, "null output handle");
        if (nbytes && !text) throw Error(FPG_EINVAL, "null text");
        const std::vector<int32_t> devs = checked_devices(devices, ndevices);
        auto t0 = std::chrono::steady_clock::now();
        auto D = new_dict(scheme, id_base, devs);
        const size_t G = devs.size();
        // Every device splits the whole text (HBM-bound, in parallel): newline
        // positions, newline-free bytes and word offsets; each keeps its range.
        std::vector<uint64_t> nwords(G, 0);
        for_each_shard(G, [&](size_t g) {
            Shard& sh = *D->shards[g];
            CK(cudaSetDevice(sh.device));
            CK(cudaStreamCreateWithFlags(&sh.stream, cudaStreamNonBlocking));
            cudaStream_t st = sh.stream;
            DBuf<uint8_t> dtext;
            dtext.reserve(nbytes + 16);
            if (nbytes) CK(cudaMemcpyAsync(dtext.p, text, nbytes, cudaMemcpyHostToDevice, st));
            sh.d_hist.reserve(256);
            sh.h_hist.reserve(256);
            byte_histogram(dtext.p, nbytes, sh.d_hist.p, st);
            CK(cudaMemcpyAsync(sh.h_hist.p, sh.d_hist.p, 256 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
            CK(cudaStreamSynchronize(st));
            const uint64_t nl = sh.h_hist.p[(unsigned char)'\n'];
            const uint64_t kept = nbytes - nl;
            const uint64_t n = nl + ((nbytes && text[nbytes - 1] != '\n') ? 1 : 0);
            DBuf<uint64_t> pos;
            DBuf<uint64_t> count;
            DBuf<uint8_t> tmp;
            pos.reserve(std::max<uint64_t>(nl, 1));
            count.reserve(1);
            sh.blob.reserve(kept + 16);
            sh.offs.reserve(n + 1);
            size_t tb = 0, tb2 = 0;
            thrust::counting_iterator<uint64_t> idx(0);
            CK(cub::DeviceSelect::If(nullptr, tb, idx, pos.p, count.p, (int64_t)nbytes, IsNewline{dtext.p}, st));
            CK(cub::DeviceSelect::If(nullptr, tb2, dtext.p, sh.blob.p, count.p, (int64_t)nbytes, NotNewline{}, st));
            tmp.reserve(std::max(tb, tb2));
            if (nbytes) {
                CK(cub::DeviceSelect::If(tmp.p, tb, idx, pos.p, count.p, (int64_t)nbytes, IsNewline{dtext.p}, st));
                CK(cub::DeviceSelect::If(tmp.p, tb2, dtext.p, sh.blob.p, count.p, (int64_t)nbytes, NotNewline{}, st));
            }
            k_text_offsets<<<(unsigned)cdiv(n + 1, 256), 256, 0, st>>>(pos.p, n, kept, sh.offs.p);
            CK(cudaGetLastError());
            CK(cudaStreamSynchronize(st));
            nwords[g] = n;
            // histogram of the words themselves (the newlines are separators)
            sh.h_hist.p[(unsigned char)'\n'] = 0;
        });
        assign_ranges(*D, nwords[0]);
        std::vector<unsigned long long> hist(256, 0);
        for (int c = 0; c < 256; ++c) hist[c] = D->shards[0]->h_hist.p[c];
        std::vector<uint64_t> offs_at(G);
        for (size_t g = 0; g < G; ++g) offs_at[g] = D->shards[g]->base;
        finish_dict(*D, hist, offs_at, t0);
        *out = D.release();
    });
}

int fpg_byte_histogram(const uint8_t* bytes, uint64_t nbytes, int32_t device, uint64_t* counts) {
    return guarded([&] {
        if (!counts || (nbytes && !bytes)) throw Error(FPG_EINVAL, "null argument");
        CK(cudaSetDevice(device));
        cudaStream_t st;
        CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
        std::unique_ptr<CUstream_st, void (*)(CUstream_st*)> guard(st, [](CUstream_st* s) { cudaStreamDestroy(s); });
        DBuf<uint8_t> d;
        DBuf<unsigned long long> h;
        d.reserve(nbytes);
        h.reserve(256);
        if (nbytes) CK(cudaMemcpyAsync(d.p, bytes, nbytes, cudaMemcpyHostToDevice, st));
        byte_histogram(d.p, nbytes, h.p, st);
        CK(cudaMemcpyAsync(counts, h.p, 256 * sizeof(uint64_t), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
    });
}

int fpg_dict_destroy(fpg_dict* dict) {
    return guarded([&] {
        if (dict && dict->live_batches.load() > 0)
            throw Error(FPG_EINVAL, "fpg_dict_destroy with live batches: destroy them first");
        delete dict;
    });
}

int fpg_dict_size(const fpg_dict* dict, uint64_t* n) {
    return guarded([&] {
        if (!dict || !n) throw Error(FPG_EINVAL, "null argument");
        *n = dict->n;
    });
}

int fpg_dict_build_seconds(const fpg_dict* dict, double* seconds) {
    return guarded([&] {
        if (!dict || !seconds) throw Error(FPG_EINVAL, "null argument");
        *seconds = dict->build_seconds;
    });
}

int fpg_dict_build_profile(const fpg_dict* dict, int32_t shard, fpg_build_stage* out, int32_t cap, int32_t* nstages) {
    return guarded([&] {
        if (!dict || !nstages || (cap > 0 && !out)) throw Error(FPG_EINVAL, "null argument");
        if (shard < 0 || shard >= (int32_t)dict->shards.size()) throw Error(FPG_EINVAL, "no such shard");
        const auto& st = dict->shards[(size_t)shard]->dict.stages;
        *nstages = (int32_t)st.size();
        for (int32_t i = 0; i < cap && i < (int32_t)st.size(); ++i) out[i] = st[(size_t)i];
    });
}

int fpg_dict_prints(const fpg_dict* dict, uint64_t* out) {
    return guarded([&] {
        if (!dict || (!out && dict->n)) throw Error(FPG_EINVAL, "null argument");
        for (auto& shp : dict->shards) {
            Shard& sh = *shp;
            if (!sh.n) continue;
            CK(cudaSetDevice(sh.device));
            DBuf<uint64_t> tmp;
            tmp.reserve(sh.n);
            fpg::k_scatter_prints<<<(unsigned)cdiv(sh.n, 256), 256, 0, sh.stream>>>(sh.dict.fp.p, sh.dict.ids.p, sh.n, tmp.p);
            CK(cudaGetLastError());
            CK(cudaMemcpyAsync(out + sh.base, tmp.p, sh.n * sizeof(uint64_t), cudaMemcpyDeviceToHost, sh.stream));
            CK(cudaStreamSynchronize(sh.stream));
        }
    });
}

int fpg_build_fingerprints(const uint8_t* bytes, const uint64_t* offsets, uint64_t n, const fpg_scheme* scheme,
                           int32_t device, uint64_t* out) {
    return guarded([&] {
        validate(scheme);
        if (n && (!offsets || !out)) throw Error(FPG_EINVAL, "null argument");
        if (n && offsets[n] > offsets[0] && !bytes) throw Error(FPG_EINVAL, "null bytes");
        CK(cudaSetDevice(device));
        if (!n) return;
        const fpg::SchemeParams P = make_params(*scheme);
        const uint64_t b0 = offsets[0], nbytes = offsets[n] - b0;
        std::vector<uint64_t> local(n + 1);
        for (uint64_t i = 0; i <= n; ++i) {
            local[i] = offsets[i] - b0;
            if (i && offsets[i] - offsets[i - 1] > (uint64_t)fpg::kMaxLen)
                throw Error(FPG_EINVAL, "string longer than FPG_MAX_WORD_LEN");
        }
        cudaStream_t st;
        CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
        std::unique_ptr<CUstream_st, void (*)(CUstream_st*)> guard(st, [](CUstream_st* s) { cudaStreamDestroy(s); });
        DBuf<uint8_t> blob;
        DBuf<uint64_t> offs, fp;
        blob.reserve(nbytes + 16);
        offs.reserve(n + 1);
        fp.reserve(n);
        if (nbytes) CK(cudaMemcpyAsync(blob.p, bytes + b0, nbytes, cudaMemcpyHostToDevice, st));
        CK(cudaMemcpyAsync(offs.p, local.data(), (n + 1) * sizeof(uint64_t), cudaMemcpyHostToDevice, st));
        const unsigned grid = (unsigned)cdiv(n, 256);
        switch (P.variant) {
            case 0: fpg::k_build<0><<<grid, 256, 0, st>>>(blob.p, offs.p, nullptr, n, nullptr, nullptr, P, fp.p, nullptr, nullptr, nullptr, nullptr, nullptr); break;
            case 1: fpg::k_build<1><<<grid, 256, 0, st>>>(blob.p, offs.p, nullptr, n, nullptr, nullptr, P, fp.p, nullptr, nullptr, nullptr, nullptr, nullptr); break;
            case 2: fpg::k_build<2><<<grid, 256, 0, st>>>(blob.p, offs.p, nullptr, n, nullptr, nullptr, P, fp.p, nullptr, nullptr, nullptr, nullptr, nullptr); break;
            default: fpg::k_build<3><<<grid, 256, 0, st>>>(blob.p, offs.p, nullptr, n, nullptr, nullptr, P, fp.p, nullptr, nullptr, nullptr, nullptr, nullptr); break;
        }
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(out, fp.p, n * sizeof(uint64_t), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
    });
}

int fpg_batch_create(fpg_dict* dict, fpg_batch** out) {
    return guarded([&] {
        if (!dict || !out) throw Error(FPG_EINVAL, "null argument");
        make_batch(dict, out);
        (*out)->external = true;
        ++dict->live_batches;
    });
}

int fpg_batch_destroy(fpg_batch* batch) {
    return guarded([&] {
        if (batch && batch->external) --batch->dict->live_batches;
        delete batch;
    });
}

int fpg_batch_upload(fpg_batch* batch, const uint8_t* qbytes, const uint64_t* qoffsets, uint64_t nq) {
    return guarded([&] {
        if (!batch) throw Error(FPG_EINVAL, "null batch");
        upload(batch, qbytes, qoffsets, nq);
        batch->ran = false;
    });
}

int fpg_batch_run(fpg_batch* batch, const fpg_query_options* opt) {
    return guarded([&] {
        if (!batch) throw Error(FPG_EINVAL, "null batch");
        run(batch, opt);
    });
}

int fpg_batch_download(fpg_batch* batch, fpg_result* out) {
    return guarded([&] {
        if (!batch || !out) throw Error(FPG_EINVAL, "null argument");
        download(batch, out);
    });
}

int fpg_batch_last_timing(const fpg_batch* batch, int32_t shard, double* run_ms, double* filter_ms,
                          uint64_t* executed_pairs, uint64_t* survivors, uint64_t* kernel_launches) {
    return guarded([&] {
        if (!batch || shard < 0 || (size_t)shard >= batch->sb.size()) throw Error(FPG_EINVAL, "bad shard");
        const ShardBatch& S = *batch->sb[(size_t)shard];
        if (run_ms) *run_ms = S.run_ms;
        if (filter_ms) *filter_ms = S.filter_ms;
        if (executed_pairs) *executed_pairs = S.executed;
        if (survivors) *survivors = S.survivors;
        if (kernel_launches) *kernel_launches = S.launches;
    });
}

int fpg_batch_last_host_ms(const fpg_batch* batch, double* upload_ms, double* download_ms, double* assemble_ms) {
    return guarded([&] {
        if (!batch) throw Error(FPG_EINVAL, "null batch");
        if (upload_ms) *upload_ms = batch->upload_ms;
        if (download_ms) *download_ms = batch->download_ms;
        if (assemble_ms) *assemble_ms = batch->assemble_ms;
    });
}

int fpg_batch_device_csr(const fpg_batch* batch, int32_t shard, int32_t* device, uint64_t* total,
                         const uint64_t** d_offsets, const uint32_t** d_ids) {
    return guarded([&] {
        if (!batch || shard < 0 || (size_t)shard >= batch->sb.size()) throw Error(FPG_EINVAL, "bad shard");
        if (!batch->ran) throw Error(FPG_EINVAL, "fpg_batch_device_csr before a successful fpg_batch_run");
        const ShardBatch& S = *batch->sb[(size_t)shard];
        if (device) *device = S.sh->device;
        if (total) *total = S.total;
        if (d_offsets) *d_offsets = S.offsets.p;
        if (d_ids) *d_ids = S.ids_out;
    });
}

int fpg_csr_merge_device(int32_t device, int32_t nparts, const uint64_t* const* d_offsets,
                         const uint32_t* const* d_ids, uint64_t nq, uint64_t* d_out_offsets, uint32_t* d_out_ids,
                         void* stream) {
    return guarded([&] {
        if (nparts < 1 || nparts > fpg::kMaxMergeParts) throw Error(FPG_EINVAL, "nparts out of range");
        if (!d_offsets || !d_ids || !d_out_offsets) throw Error(FPG_EINVAL, "null argument");
        CK(cudaSetDevice(device));
        cudaStream_t st = static_cast<cudaStream_t>(stream);
        fpg::MergeParts mp{};
        mp.n = nparts;
        for (int i = 0; i < nparts; ++i) {
            if (!d_offsets[i]) throw Error(FPG_EINVAL, "null part offsets");
            mp.off[i] = d_offsets[i];
            mp.ids[i] = d_ids[i];
        }
        // row lengths summed over the parts (+ a zero at nq), then their
        // exclusive scan: the merged offsets
        size_t tmp = 0;
        CK(cub::DeviceScan::ExclusiveSum(nullptr, tmp, d_out_offsets, d_out_offsets, nq + 1, st));
        const size_t cnt_bytes = ((nq + 1) * sizeof(uint64_t) + 255) & ~size_t(255);
        uint8_t* d_tmp = nullptr;
        CK(cudaMallocAsync(reinterpret_cast<void**>(&d_tmp), cnt_bytes + std::max<size_t>(tmp, 1), st));
        uint64_t* d_cnt = reinterpret_cast<uint64_t*>(d_tmp);
        const unsigned blocks = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(cdiv(nq + 1, 256), 148 * 16));
        fpg::k_merge_counts<<<blocks, 256, 0, st>>>(mp, nq, d_cnt);
        CK(cudaGetLastError());
        CK(cub::DeviceScan::ExclusiveSum(d_tmp + cnt_bytes, tmp, d_cnt, d_out_offsets, nq + 1, st));
        CK(cudaFreeAsync(d_tmp, st));
        if (nq) {
            fpg::k_merge_rows<<<(unsigned)std::min<uint64_t>(cdiv(nq * 32, 256), 148 * 16), 256, 0, st>>>(
                mp, nq, d_out_offsets, d_out_ids);
            CK(cudaGetLastError());
        }
        g_launches += 4;
    });
}

int fpg_dict_scan_shape(const fpg_dict* dict, int32_t* sliced, int32_t* sig_fields) {
    return guarded([&] {
        if (!dict || !sliced || !sig_fields) throw Error(FPG_EINVAL, "null argument");
        *sliced = dict->slice ? 1 : 0;
        *sig_fields = dict->params.nsig;
    });
}

int fpg_batch_last_candidates(const fpg_batch* batch, int32_t shard, uint64_t* candidates) {
    return guarded([&] {
        if (!batch || !candidates || shard < 0 || (size_t)shard >= batch->sb.size()) throw Error(FPG_EINVAL, "bad shard");
        *candidates = batch->sb[(size_t)shard]->candidates;
    });
}

int fpg_batch_last_verify(const fpg_batch* batch, int32_t shard, double* verify_ms, uint64_t* records,
                          uint32_t* rounds, double* plan_ms) {
    return guarded([&] {
        if (!batch || shard < 0 || (size_t)shard >= batch->sb.size()) throw Error(FPG_EINVAL, "bad shard");
        const ShardBatch& S = *batch->sb[(size_t)shard];
        if (verify_ms) *verify_ms = S.verify_ms;
        if (plan_ms) *plan_ms = S.plan_ms;
        if (records) *records = S.cand_records;
        if (rounds) *rounds = S.cand_rounds;
    });
}

int fpg_batch_last_scanned(const fpg_batch* batch, int32_t shard, uint64_t* scanned) {
    return guarded([&] {
        if (!batch || !scanned || shard < 0 || (size_t)shard >= batch->sb.size()) throw Error(FPG_EINVAL, "bad shard");
        *scanned = batch->sb[(size_t)shard]->scanned;
    });
}

int fpg_batch_last_scanned_exact(const fpg_batch* batch, int32_t shard, uint64_t* scanned) {
    return guarded([&] {
        if (!batch || !scanned || shard < 0 || (size_t)shard >= batch->sb.size()) throw Error(FPG_EINVAL, "bad shard");
        *scanned = batch->sb[(size_t)shard]->scanned_x;
    });
}

int fpg_query_batch(fpg_dict* dict, const uint8_t* qbytes, const uint64_t* qoffsets, uint64_t nq,
                    const fpg_query_options* opt, fpg_result* out) {
    return guarded([&] {
        if (!dict || !out) throw Error(FPG_EINVAL, "null argument");
        check_opts(dict, opt);
        // An idle scratch batch from the dictionary's pool (a new one when all
        // are busy); concurrent callers get separate batches and streams.
        fpg_batch* b = nullptr;
        {
            std::lock_guard<std::mutex> lk(dict->cache_mu);
            if (!dict->pool.empty()) {
                b = dict->pool.back();
                dict->pool.pop_back();
            }
        }
        if (!b) make_batch(dict, &b);
        std::unique_ptr<fpg_batch> own(b);
        upload(b, qbytes, qoffsets, nq, false);
        run(b, opt);
        download(b, out);
        std::lock_guard<std::mutex> lk(dict->cache_mu);
        if (dict->pool.size() < 16) dict->pool.push_back(own.release());
    });
}

int fpg_result_free(fpg_result* res) {
    return guarded([&] {
        if (!res) return;
        PinnedPool& pool = pinned_pool();
        for (void* p : {(void*)res->offsets, (void*)res->word_ids, (void*)res->stats})
            if (!pool.put(p)) std::free(p);
        std::memset(res, 0, sizeof(*res));
    });
}

}  // extern "C"
