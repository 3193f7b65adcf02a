// ALU / FMA integer pipe peaks on sm_100a: the denominators of K2's roofline.
//
// Each thread runs C independent dependency chains; the loop body is U
// unrolled rounds of one instruction per chain, written as inline PTX so
// the SASS is exactly that instruction (check: cuobjdump -sass alupipe |
// grep -c LOP3 etc., printed by alupipe.sh).  Loop overhead is 3
// instructions per C*U = 512 counted ones (< 0.6%).  Kernels:
//   LOP3        lop3.b32 (ALU pipe)
//   IMAD        mad.lo.u32 (FMA pipe)
//   LOP3+IMAD   alternating, C/2 chains of each (dual issue: ALU + FMA)
//   LOP3x2+IMAD two LOP3 per IMAD (K2's mix is ~1.7 : 1)
// Reported: warp instructions per clock per SM, and thread ops per clock
// per SM (x32), from CUDA-event time x the SM clock read by NVML-free
// clock64 sampling (sm clock = clock64 delta / event time).
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

constexpr int C = 16;   // chains per thread
constexpr int U = 32;   // unrolled rounds per loop iteration

__device__ __forceinline__ uint32_t lop(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t d;
    asm volatile("lop3.b32 %0, %1, %2, %3, 0x96;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    return d;
}
__device__ __forceinline__ uint32_t mad(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t d;
    asm volatile("mad.lo.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    return d;
}

// MODE 0: LOP3 only; 1: IMAD only; 2: alternate; 3: LOP3, LOP3, IMAD
template <int MODE>
__global__ void __launch_bounds__(256) kern(uint32_t* out, uint32_t s, uint32_t m, int iters, long long* clk) {
    uint32_t v[C];
#pragma unroll
    for (int i = 0; i < C; ++i) v[i] = threadIdx.x * 0x9e3779b9u + i;
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
            for (int i = 0; i < C; ++i) {
                if (MODE == 0) v[i] = lop(v[i], s, m);
                else if (MODE == 1) v[i] = mad(v[i], s, m);
                else if (MODE == 2) v[i] = (i & 1) ? mad(v[i], s, m) : lop(v[i], s, m);
                else v[i] = (i % 3 == 2) ? mad(v[i], s, m) : lop(v[i], s, m);
            }
    }
    const long long t1 = clock64();
    uint32_t r = 0;
#pragma unroll
    for (int i = 0; i < C; ++i) r ^= v[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = r;
    if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}

template <int MODE>
void run(const char* name, int blocks, uint32_t* d_out, long long* d_clk, int sms) {
    const int threads = 256, iters = 2048;
    kern<MODE><<<blocks, threads>>>(d_out, 0x12345678u, 0x9abcdef0u, 64, d_clk);  // warm-up
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
        cudaEventRecord(a);
        kern<MODE><<<blocks, threads>>>(d_out, 0x12345678u, 0x9abcdef0u, iters, d_clk);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (ms < best) best = ms;
    }
    long long c0 = 0;
    cudaMemcpy(&c0, d_clk, sizeof(c0), cudaMemcpyDeviceToHost);
    const double warp_instr = (double)blocks * (threads / 32) * iters * U * C;
    const double mhz = c0 / (best * 1e3);  // block 0's clock span over the launch time (upper bound of its share)
    const double per_sm_s = warp_instr / sms / (best * 1e-3);
    printf("%-12s blocks=%d  ms=%.3f  thread-ops/s=%.4e  warp-instr/s/SM=%.4e  block0_clk_MHz~%.0f\n", name, blocks,
           best, warp_instr * 32 / (best * 1e-3), per_sm_s, mhz);
}

int main() {
    cudaDeviceProp p;
    cudaGetDeviceProperties(&p, 0);
    int clk_khz = 0;
    cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
    printf("device %s SMs=%d clockRate(kHz)=%d\n", p.name, p.multiProcessorCount, clk_khz);
    const int sms = p.multiProcessorCount;
    uint32_t* d_out;
    long long* d_clk;
    const int blocks = sms * 8;  // 8 x 256 threads = 64 warps per SM, one wave
    cudaMalloc(&d_out, sizeof(uint32_t) * blocks * 256);
    cudaMalloc(&d_clk, sizeof(long long) * blocks);
    run<0>("LOP3", blocks, d_out, d_clk, sms);
    run<1>("IMAD", blocks, d_out, d_clk, sms);
    run<2>("LOP3+IMAD", blocks, d_out, d_clk, sms);
    run<3>("2LOP3+IMAD", blocks, d_out, d_clk, sms);
    for (int w : {1, 2, 4}) {  // fewer warps per SM: the occupancy K2 runs at
        printf("-- %d block(s) of 8 warps per SM\n", w);
        run<0>("LOP3", sms * w, d_out, d_clk, sms);
        run<3>("2LOP3+IMAD", sms * w, d_out, d_clk, sms);
    }
    const cudaError_t e = cudaDeviceSynchronize();
    printf("status %s\n", cudaGetErrorString(e));
    return e == cudaSuccess ? 0 : 1;
}
