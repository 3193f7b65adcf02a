// fpg_host.h -- host-side pieces shared by the translation units of libfpg.so:
// the error type every C-ABI entry point converts to a status code, the CK
// check of CUDA runtime calls, and the K2 launchers compiled in their own
// translation units (fpg_k2_*.cu, so nvcc builds the many template
// instantiations in parallel).
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <stdexcept>
#include <string>

#include "../../include/fpg.h"
#include "fpg_kernels.cuh"

namespace fpg_host {

struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

}  // namespace fpg_host

#define CK(x)                                                                                  \
    do {                                                                                       \
        cudaError_t e_ = (x);                                                                  \
        if (e_ != cudaSuccess)                                                                 \
            throw fpg_host::Error(FPG_ECUDA, std::string(#x) + ": " + cudaGetErrorString(e_) + \
                                                 " (" + __FILE__ + ":" + std::to_string(__LINE__) + ")"); \
    } while (0)

namespace fpg_host {

// K2 bit-sliced (fpg_k2_slice_w{16,32,64}.cu): k_slice<W, fw, extra, nsig>.
void dispatch_slice_16(int fw, int nsig, const fpg::SliceTile* tiles, uint32_t ntiles, const fpg::SliceParams& P,
                       cudaStream_t st, int device);
void dispatch_slice_32(int fw, int nsig, const fpg::SliceTile* tiles, uint32_t ntiles, const fpg::SliceParams& P,
                       cudaStream_t st, int device);
void dispatch_slice_64(int fw, int nsig, const fpg::SliceTile* tiles, uint32_t ntiles, const fpg::SliceParams& P,
                       cudaStream_t st, int device);
// exact Hamming path of words <= kXLen bytes, W = 16 (fpg_k2_slice_w16.cu)
void dispatch_slice_16x(int fw, const fpg::SliceTile* tiles, uint32_t ntiles, const fpg::SliceParams& P,
                        cudaStream_t st, int device);
// K2 generic (fpg_k2_scan.cu): k_scan<kind, W, stats>.
void dispatch_scan(int kind, int width, bool stats, const fpg::Tile* tiles, uint32_t ntiles,
                   const fpg::ScanParams& P, cudaStream_t st, int device);

}  // namespace fpg_host
