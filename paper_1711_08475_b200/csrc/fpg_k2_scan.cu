// fpg_k2_scan.cu -- instantiations and launcher of the generic K2, k_scan
// (fpg_scan.cuh), in their own translation unit (parallel nvcc builds).
#define FPG_K2_TU
#include "fpg_host.h"

namespace fpg_host {
namespace {

template <int KIND, int W, bool STATS>
void launch_scan(const fpg::Tile* tiles, uint32_t ntiles, const fpg::ScanParams& P, cudaStream_t st,
                 int device) {
    auto kern = fpg::k_scan<KIND, W, STATS>;
    constexpr size_t smem = fpg::scan_smem_bytes(W, STATS);
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    int per_sm = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, fpg::kScanThreads, smem));
    const uint64_t grid = std::min<uint64_t>(ntiles, (uint64_t)sms * std::max(per_sm, 1) * 8);
    kern<<<(unsigned)std::max<uint64_t>(grid, 1), fpg::kScanThreads, smem, st>>>(tiles, ntiles, P);
    CK(cudaGetLastError());
}

template <int KIND>
void launch_w(int width, bool stats, const fpg::Tile* tiles, uint32_t ntiles, const fpg::ScanParams& P,
              cudaStream_t st, int device) {
    if (width == 16) stats ? launch_scan<KIND, 16, true>(tiles, ntiles, P, st, device)
                           : launch_scan<KIND, 16, false>(tiles, ntiles, P, st, device);
    else if (width == 32) stats ? launch_scan<KIND, 32, true>(tiles, ntiles, P, st, device)
                                : launch_scan<KIND, 32, false>(tiles, ntiles, P, st, device);
    else stats ? launch_scan<KIND, 64, true>(tiles, ntiles, P, st, device)
               : launch_scan<KIND, 64, false>(tiles, ntiles, P, st, device);
}

}  // namespace

void dispatch_scan(int kind, int width, bool stats, const fpg::Tile* tiles, uint32_t ntiles,
                   const fpg::ScanParams& P, cudaStream_t st, int device) {
    switch (kind) {
        case fpg::kPopc: launch_w<fpg::kPopc>(width, stats, tiles, ntiles, P, st, device); break;
        case fpg::kFold2: launch_w<fpg::kFold2>(width, stats, tiles, ntiles, P, st, device); break;
        case fpg::kFold4: launch_w<fpg::kFold4>(width, stats, tiles, ntiles, P, st, device); break;
        case fpg::kPos3: launch_w<fpg::kPos3>(width, stats, tiles, ntiles, P, st, device); break;
        default: launch_w<fpg::kGeneric>(width, stats, tiles, ntiles, P, st, device); break;
    }
}

}  // namespace fpg_host
