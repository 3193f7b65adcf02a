// LOP3 issue rate with three distinct register sources per instruction (the
// carry-save adder's operand pattern in K2) vs the same-source pattern of
// alupipe.cu, at 16 and 32 warps per SM.  Prints LOP3 thread-ops/clk/SM.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

constexpr int C = 12;
template <int LUT>
__device__ __forceinline__ uint32_t lop(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t d;
    asm volatile("lop3.b32 %0, %1, %2, %3, %4;" : "=r"(d) : "r"(a), "r"(b), "r"(c), "n"(LUT));
    return d;
}

// MODE 0: v = lop(v, s, m) (shared sources); 1: three distinct registers per LOP3
// (full adders over rotating chain state, as in the counter)
template <int MODE>
__global__ void kern(uint32_t* out, uint32_t s, uint32_t m, int iters) {
    uint32_t a[C], b[C];
#pragma unroll
    for (int i = 0; i < C; ++i) { a[i] = threadIdx.x * 0x9e3779b9u + i; b[i] = a[i] ^ 0x5bd1e995u; }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < 16; ++u)
#pragma unroll
            for (int i = 0; i < C; ++i) {
                if (MODE == 0) {
                    a[i] = lop<0x96>(a[i], s, m);
                    b[i] = lop<0xe8>(b[i], s, m);
                } else if (MODE == 2) {  // K2's mix: LOP3 on a, IMAD on b (FMA pipe)
                    a[i] = lop<0x96>(a[i], s, m);
                    asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(b[i]) : "r"(s), "r"(m));
                } else if (MODE == 3) {  // two LOP3 per IMAD
                    a[i] = lop<0x96>(a[i], s, m);
                    if (i % 2) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(b[i]) : "r"(s), "r"(m));
                    else b[i] = lop<0xe8>(b[i], s, m);
                } else {
                    const uint32_t x = a[(i + 1) % C], y = b[(i + 5) % C];
                    const uint32_t na = lop<0x96>(a[i], x, y);
                    b[i] = lop<0xe8>(b[i], x, y);
                    a[i] = na;
                }
            }
    }
    uint32_t r = 0;
#pragma unroll
    for (int i = 0; i < C; ++i) r ^= a[i] ^ b[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}

template <int MODE>
void run(const char* name, int per_sm, int sms, uint32_t* d) {
    const int threads = 256, blocks = sms * per_sm, iters = 1024;
    kern<MODE><<<blocks, threads>>>(d, 1, 2, 16);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(e0);
        kern<MODE><<<blocks, threads>>>(d, 1, 2, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        best = ms < best ? ms : best;
    }
    int khz = 0;
    cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, 0);
    const double ops = (double)blocks * threads * iters * 16 * C * (MODE == 2 ? 1 : MODE == 3 ? 1.5 : 2);
    printf("%-22s warps/SM=%2d  LOP3 thread-ops/clk/SM = %.2f (at %d MHz)\n", name, per_sm * 8,
           ops / (best * 1e-3) / sms / (khz * 1e3), khz / 1000);
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    uint32_t* d;
    cudaMalloc(&d, 1 << 24);
    for (int per_sm : {1, 2, 3, 4, 8}) {
        run<0>("shared sources", per_sm, sms, d);
        run<1>("distinct sources", per_sm, sms, d);
        run<2>("LOP3+IMAD (LOP3 rate)", per_sm, sms, d);
        run<3>("2 LOP3+IMAD (LOP3 rate)", per_sm, sms, d);
    }
    printf("status %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
}
