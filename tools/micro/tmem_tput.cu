// Microbenchmark: tcgen05.ld (32x32b.x32) and tcgen05.st throughput per SM (perf experiment only).
#include <cstdio>
#include <stdint.h>
#include "../../paper_2604_21221_b200/csrc/ptx.cuh"
using namespace pbsa;

template <int WARPS, int MODE>
__global__ void __launch_bounds__(WARPS * 32) k(uint32_t* out, int iters) {
    __shared__ uint32_t holder;
    const int warp = threadIdx.x >> 5;
    if (warp == 0) tmem_alloc<256>(&holder);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = holder + ((static_cast<uint32_t>(warp & 3) * 32) << 16);
    uint32_t acc = 0;
    uint32_t r[32];
    for (int c = 0; c < 32; ++c) r[c] = c;
    for (int it = 0; it < iters; ++it) {
        const uint32_t col = ((it + warp) & 7) * 32;
        if (MODE == 0) {
            tmem_ld32(tmem + col, r);
            tmem_wait_ld();
#pragma unroll
            for (int c = 0; c < 32; c += 2) acc ^= r[c] + r[c + 1];
        } else if (MODE == 1) {
            uint32_t a[32], b[32];
            tmem_ld32(tmem + col, a);
            tmem_ld32(tmem + ((col + 32) & 255), b);
            tmem_wait_ld();
#pragma unroll
            for (int c = 0; c < 32; ++c) acc ^= a[c] + b[c];
        } else {
            r[0] = it;
            tmem_st32(tmem + col, r);
            tmem_wait_st();
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc<256>(holder);
}

template <int WARPS, int MODE>
void run(const char* name, int ctas_per_sm) {
    uint32_t* out;
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaMalloc(&out, 4 * sms * ctas_per_sm * WARPS * 32);
    const int iters = 20000;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0);
        k<WARPS, MODE><<<sms * ctas_per_sm, WARPS * 32>>>(out, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
    }
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    int clk;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const double per_ld = (MODE == 1 ? 2 : 1) * 32.0 * 32 * 4;
    const double bytes = double(sms) * ctas_per_sm * WARPS * iters * per_ld;
    const double cyc = ms * 1e-3 * clk * 1e3;
    printf("%-28s warps/CTA %d CTAs/SM %d: %.1f B/clk/SM (%.3f ms, err %s)\n", name, WARPS, ctas_per_sm,
           bytes / cyc / sms, ms, cudaGetErrorString(cudaGetLastError()));
    cudaFree(out);
}

int main() {
    run<4, 0>("ld x32 + wait", 1);
    run<4, 0>("ld x32 + wait", 2);
    run<8, 0>("ld x32 + wait", 1);
    run<8, 0>("ld x32 + wait", 2);
    run<4, 1>("2x ld x32 + wait", 1);
    run<4, 1>("2x ld x32 + wait", 2);
    run<8, 1>("2x ld x32 + wait", 2);
    run<4, 2>("st x32 + wait", 2);
    run<8, 2>("st x32 + wait", 2);
    return 0;
}
