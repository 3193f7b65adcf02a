// Phase-0 microbenchmark: per-SM issue rates of the integer ops the filter uses
// (LOP3, IADD3, POPC, FLO) on sm_100a, measured with clock64 over a dependent-free
// unrolled loop. Prints ops/clk/SM for each. Not part of the product.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define ITERS 4096
#define ILP 8

template <int OP>
__global__ void kern(uint32_t* out, uint32_t seed, long long* clk) {
    uint32_t v[ILP];
#pragma unroll
    for (int i = 0; i < ILP; ++i) v[i] = seed * (threadIdx.x + 1) + i * 0x9e3779b9u;
    uint32_t acc = 0;
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int i = 0; i < ILP; ++i) {
            if (OP == 0) { v[i] = (v[i] ^ seed) & (v[i] | it); }              // LOP3
            else if (OP == 1) { v[i] = v[i] + seed + it; }                   // IADD3
            else if (OP == 2) { v[i] = __popc(v[i]) + v[i]; }                // POPC (+IADD)
            else if (OP == 3) { v[i] = __clz(v[i]) ^ v[i]; }                 // FLO (+LOP)
            else if (OP == 4) { uint32_t x = v[i] ^ seed; acc += (__popc(x) < 3); v[i] += 1; } // filter idiom
        }
    }
    long long t1 = clock64();
    uint32_t r = acc;
#pragma unroll
    for (int i = 0; i < ILP; ++i) r ^= v[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = r;
    if (threadIdx.x == 0 && blockIdx.x == 0) *clk = t1 - t0;
}

template <int OP>
void run(const char* name, int blocks, int threads, uint32_t* d_out, long long* d_clk) {
    kern<OP><<<blocks, threads>>>(d_out, 12345, d_clk);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    kern<OP><<<blocks, threads>>>(d_out, 12345, d_clk);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    long long clk; cudaMemcpy(&clk, d_clk, sizeof(clk), cudaMemcpyDeviceToHost);
    int dev; cudaGetDevice(&dev); cudaDeviceProp p; cudaGetDeviceProperties(&p, dev);
    double ops = (double)blocks * threads * ITERS * ILP;
    double per_sm_clk = ops / p.multiProcessorCount / (double)clk;  // block 0's clock span
    printf("%-8s blocks=%d threads=%d ms=%.3f  elem-ops/s=%.3e  elem-ops/clk/SM(block0 span)=%.2f  eff_clock_MHz=%.0f\n",
           name, blocks, threads, ms, ops / (ms * 1e-3), per_sm_clk, clk / (ms * 1e3));
}

int main() {
    cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
    printf("device %s SMs=%d clock(kHz)=%d\n", p.name, p.multiProcessorCount, p.clockRate);
    uint32_t* d_out; long long* d_clk;
    int blocks = p.multiProcessorCount * 4, threads = 512;
    cudaMalloc(&d_out, sizeof(uint32_t) * blocks * threads);
    cudaMalloc(&d_clk, sizeof(long long));
    run<0>("LOP3", blocks, threads, d_out, d_clk);
    run<1>("IADD3", blocks, threads, d_out, d_clk);
    run<2>("POPC+ADD", blocks, threads, d_out, d_clk);
    run<3>("FLO+LOP", blocks, threads, d_out, d_clk);
    run<4>("FILTER", blocks, threads, d_out, d_clk);
    cudaError_t e = cudaDeviceSynchronize();
    printf("status %s\n", cudaGetErrorString(e));
    return 0;
}
