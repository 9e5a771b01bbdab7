// Microbenchmark: tcgen05.mma issue throughput per shape / operand source (perf experiment only).
// One CTA per SM, one elected thread issues `iters` x 8 MMAs back to back, commit + wait, clock64.
#include <cstdio>
#include <stdint.h>
#include "../../paper_2604_21221_b200/csrc/ptx.cuh"
using namespace pbsa;

// A reused through the collector buffer: fill on the first of two MMAs, lastuse on the second
__device__ __forceinline__ void mma_ss_col(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc, int fill) {
    if (fill)
        asm volatile("{ .reg .pred p; setp.ne.b32 p, 1, 0;\n"
                     "tcgen05.mma.cta_group::1.kind::f16.collector::a::fill [%0], %1, %2, %3, p; }" ::"r"(d_tmem),
                     "l"(a_desc), "l"(b_desc), "r"(idesc) : "memory");
    else
        asm volatile("{ .reg .pred p; setp.ne.b32 p, 1, 0;\n"
                     "tcgen05.mma.cta_group::1.kind::f16.collector::a::lastuse [%0], %1, %2, %3, p; }" ::"r"(d_tmem),
                     "l"(a_desc), "l"(b_desc), "r"(idesc) : "memory");
}

// TS = 2: pairs of SS MMAs sharing A (different B, different D), A through the collector;
// TS = 3: the same pairs without the collector
template <int N, int TS>
__global__ void k(long long* out, int iters) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint64_t bar;
    __shared__ uint32_t holder;
    const int warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < 65536 / 16; i += blockDim.x) reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
    if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
    if (warp == 0) tmem_alloc<512>(&holder);
    fence_proxy_async_smem();
    tc_fence_before(); __syncthreads(); tc_fence_after();
    const uint32_t tmem = holder;
    if (warp == 0) {
        const uint64_t adesc = smem_desc_sw128(smem_u32(smem), 16, 1024);
        const uint64_t bdesc = smem_desc_sw128(smem_u32(smem + 32768), 16, 1024);
        constexpr uint32_t idesc = idesc_bf16_f32(128, N, 0, 0);
        long long t0 = clock64();
        if (elect_one()) {
            for (int it = 0; it < iters; ++it) {
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) {
                    const uint64_t b2 = bdesc + (8192 >> 4);
                    if (TS == 2) {
                        mma_ss_col(tmem + 256 - 64 * (kk & 1), adesc + (((kk >> 1) * 32) >> 4), (kk & 1 ? b2 : bdesc) + (((kk >> 1) * 32) >> 4), idesc, !(kk & 1));
                    } else if (TS == 3) {
                        mma_ss(tmem + 256 - 64 * (kk & 1), adesc + (((kk >> 1) * 32) >> 4), (kk & 1 ? b2 : bdesc) + (((kk >> 1) * 32) >> 4), idesc, 1u);
                    } else if (TS) mma_ts(tmem + 256, tmem + 448 + kk * 8 % 64, bdesc + (((kk & 3) * 32) >> 4), idesc, 1u);
                    else mma_ss(tmem + 256, adesc + (((kk & 3) * 32) >> 4), bdesc + (((kk & 3) * 32) >> 4), idesc, 1u);
                }
            }
            mma_commit(&bar);
        }
        __syncwarp();
        mbar_wait(&bar, 0);
        long long t1 = clock64();
        if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
    }
    tc_fence_before(); __syncthreads();
    if (warp == 0) { tc_fence_after(); tmem_dealloc<512>(tmem); }
}

template <int N, int TS>
void run(const char* name) {
    long long* out; cudaMalloc(&out, 148 * 8);
    const int iters = 2000;
    cudaFuncSetAttribute(k<N, TS>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
    k<N, TS><<<148, 128, 65536>>>(out, iters);
    k<N, TS><<<148, 128, 65536>>>(out, iters);
    cudaDeviceSynchronize();
    long long h[148]; cudaMemcpy(h, out, sizeof(h), cudaMemcpyDeviceToHost);
    double avg = 0; for (int i = 0; i < 148; ++i) avg += h[i]; avg /= 148;
    printf("%-22s N=%3d: %.1f cycles per MMA (floor 128*N/256 = %d)  err=%s\n", name, N, avg / (iters * 8.0), N / 2,
           cudaGetErrorString(cudaGetLastError()));
    cudaFree(out);
}

int main() {
    run<64, 0>("SS M128 K16");
    run<128, 0>("SS M128 K16");
    run<256, 0>("SS M128 K16");
    run<64, 2>("SS pairs, A collector");
    run<64, 3>("SS pairs, no collector");
    run<128, 2>("SS pairs, A collector");
    run<64, 1>("TS M128 K16");
    run<128, 1>("TS M128 K16");
    run<256, 1>("TS M128 K16");
    return 0;
}
