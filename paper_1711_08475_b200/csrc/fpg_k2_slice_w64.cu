// fpg_k2_slice_w64.cu -- instantiations and launcher of the bit-sliced K2,
// k_slice<64, fw, extra, nsig> (fpg_slice.cuh), in their own translation unit
// (parallel nvcc builds).
#define FPG_K2_TU
#include "fpg_host.h"

namespace fpg_host {
namespace {

template <int NP, int FW, int EXTRA, int S>
void launch_slice(const fpg::SliceTile* tiles, uint32_t ntiles, const fpg::SliceParams& P, cudaStream_t st,
                  int device) {
    constexpr bool X = false;  // the exact path is W = 16 only
    // the common options (filter + stats + window on, k = 1) run the HOT
    // instantiation; small batches (P.no_barrier) the barrier-free one when
    // its double-buffered query data fits
    // (W = 16: HOT has no survivor counters, the histograms give the stats)
    const bool hot = P.use_fp && (NP <= 16 ? !P.stats : P.stats != 0) && P.wskip && !P.exhaustive && P.k == 1;
    constexpr bool kCanNB = fpg::slice_no_barrier(NP + S);
    const bool nb = kCanNB && P.no_barrier;
    using Kern = void (*)(const fpg::SliceTile*, uint32_t, const fpg::SliceParams);
    Kern kern;
    if constexpr (kCanNB)
        kern = nb ? (hot ? fpg::k_slice<NP, FW, EXTRA, S, true, X, true> : fpg::k_slice<NP, FW, EXTRA, S, false, X, true>)
                  : (hot ? fpg::k_slice<NP, FW, EXTRA, S, true, X, false> : fpg::k_slice<NP, FW, EXTRA, S, false, X, false>);
    else
        kern = hot ? fpg::k_slice<NP, FW, EXTRA, S, true, X, false> : fpg::k_slice<NP, FW, EXTRA, S, false, X, false>;
    const size_t smem = fpg::slice_smem_bytes(NP + S, nb);
    static int resident[2][2][64] = {{{0}}};  // per variant and device: CTAs resident on the whole GPU (0 = not queried)
    (void)X;
    const int dv = device & 63;
    if (!resident[hot][nb][dv]) {
        CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        int sms = 148, per_sm = 0;
        CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, fpg::kSliceThreads, smem));
        resident[hot][nb][dv] = sms * std::max(per_sm, 1);
    }
    const uint64_t grid = std::min<uint64_t>(ntiles, (uint64_t)resident[hot][nb][dv]);
    kern<<<(unsigned)std::max<uint64_t>(grid, 1), fpg::kSliceThreads, smem, st>>>(tiles, ntiles, P);
    CK(cudaGetLastError());
}

template <int NP, int FW, int EXTRA>
void launch_slice_s(int nsig, const fpg::SliceTile* tiles, uint32_t ntiles, const fpg::SliceParams& P,
                    cudaStream_t st, int device) {
    switch (nsig) {
        case 0: launch_slice<NP, FW, EXTRA, 0>(tiles, ntiles, P, st, device); break;
        case 8: launch_slice<NP, FW, EXTRA, 8>(tiles, ntiles, P, st, device); break;
        case 10: launch_slice<NP, FW, EXTRA, 10>(tiles, ntiles, P, st, device); break;
        case 12: launch_slice<NP, FW, EXTRA, 12>(tiles, ntiles, P, st, device); break;
        default: launch_slice<NP, FW, EXTRA, 16>(tiles, ntiles, P, st, device); break;
    }
}

}  // namespace

void dispatch_slice_64(int fw, int nsig, const fpg::SliceTile* tiles, uint32_t ntiles, const fpg::SliceParams& P,
                       cudaStream_t st, int device) {
    switch (fw) {
        case 1: launch_slice_s<64, 1, 0>(nsig, tiles, ntiles, P, st, device); break;
        case 2: launch_slice_s<64, 2, 0>(nsig, tiles, ntiles, P, st, device); break;
        case 3: launch_slice_s<64, 3, 64 % 3>(nsig, tiles, ntiles, P, st, device); break;
        default: launch_slice_s<64, 4, 0>(nsig, tiles, ntiles, P, st, device); break;
    }
}

}  // namespace fpg_host
