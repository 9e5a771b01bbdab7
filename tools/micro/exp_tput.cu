// Microbenchmark: throughput of exp2 variants on one B200 SM-set (perf experiment only).
#include <cstdio>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <stdint.h>

__device__ __forceinline__ float ex2f(float x) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ uint32_t ex2h2(uint32_t x) { uint32_t y; asm volatile("ex2.approx.f16x2 %0, %1;" : "=r"(y) : "r"(x)); return y; }
__device__ __forceinline__ uint32_t ex2b2(uint32_t x) { uint32_t y; asm volatile("ex2.approx.ftz.bf16x2 %0, %1;" : "=r"(y) : "r"(x)); return y; }
// Cody-Waite + degree-3 minimax on [0,1): 2^x = 2^i * p(f)
__device__ __forceinline__ float ex2poly(float x) {
    x = fmaxf(x, -127.f);
    float r = __fadd_rd(x, 0.f);
    float fi = floorf(x);
    float f = x - fi;
    float p = fmaf(fmaf(fmaf(0.0790199f, f, 0.2243748f), f, 0.6964755f), f, 1.0f);
    int i = __float2int_rz(fi);
    (void)r;
    return __int_as_float(__float_as_int(p) + (i << 23));
}

template <int MODE>
__global__ void k(float* out, int iters) {
    float a[8];
    for (int i = 0; i < 8; ++i) a[i] = -0.001f * (threadIdx.x + i);
    uint32_t h[8];
    for (int i = 0; i < 8; ++i) h[i] = 0xBC00BC00u ^ (threadIdx.x + i);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (MODE == 0) a[i] = ex2f(a[i]) - 1.0f;
            if (MODE == 1) h[i] = ex2h2(h[i]) ^ 0x80008000u;
            if (MODE == 2) h[i] = ex2b2(h[i]) ^ 0x80008000u;
            if (MODE == 3) a[i] = ex2poly(a[i]) - 1.0f;
        }
    }
    float s = 0;
    for (int i = 0; i < 8; ++i) s += a[i] + __uint_as_float(h[i]);
    if (s == 1234.5f) out[0] = s;
}

int main() {
    float* out; cudaMalloc(&out, 4);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int iters = 4096, threads = 512, blocks = sms * 4;
    const char* names[4] = {"ex2.f32", "ex2.f16x2", "ex2.bf16x2", "poly3.f32"};
    const double elems_per_op[4] = {1, 2, 2, 1};
    for (int mode = 0; mode < 4; ++mode) {
        cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(e0);
            if (mode == 0) k<0><<<blocks, threads>>>(out, iters);
            if (mode == 1) k<1><<<blocks, threads>>>(out, iters);
            if (mode == 2) k<2><<<blocks, threads>>>(out, iters);
            if (mode == 3) k<3><<<blocks, threads>>>(out, iters);
            cudaEventRecord(e1); cudaEventSynchronize(e1);
        }
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
        double ops = double(blocks) * threads * iters * 8;
        double per_clk_sm = ops / (ms * 1e-3) / (clk * 1e3) / sms;
        printf("%-12s %.3f ms  %.1f ops/clk/SM (at max clock %d MHz)  elems/clk/SM %.1f\n", names[mode], ms, per_clk_sm, clk / 1000, per_clk_sm * elems_per_op[mode]);
    }
    return 0;
}
