// Microbenchmark: L2 -> shared memory bulk-copy throughput per SM (perf experiment only).
// K3 streams one 16 KB K box and one 16 KB V box per visible block per CTA; at config 2 that is
// ~5.7 GB of L2 -> SM traffic per launch.  This measures what the chip delivers for that pattern:
// CTAs (1 or 2 per SM) each keep RING 16 KB bulk copies in flight from an L2-resident source.
#include <cstdio>
#include <stdint.h>
#include "../../paper_2604_21221_b200/csrc/ptx.cuh"
using namespace pbsa;

template <int RING>
__global__ void __launch_bounds__(32) k(const uint8_t* src, size_t src_bytes, int iters, uint32_t* out) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t bars[RING];
    constexpr uint32_t kBox = 16384;
    if (threadIdx.x == 0) {
        for (int s = 0; s < RING; ++s) mbar_init(bars + s, 1);
        fence_barrier_init();
    }
    __syncthreads();
    const size_t nbox = src_bytes / kBox;
    uint32_t acc = 0;
    if (threadIdx.x == 0) {
        for (int it = 0; it < iters + RING; ++it) {
            const int s = it % RING;
            if (it >= RING) {
                mbar_wait(bars + s, ((it / RING) - 1) & 1);
                acc += smem[s * kBox + (it & 1023)];
            }
            if (it < iters) {
                const size_t box = (static_cast<size_t>(blockIdx.x) * 7919 + static_cast<size_t>(it) * 131) % nbox;
                mbar_arrive_expect_tx(bars + s, kBox);
                bulk_g2s(smem + s * kBox, src + box * kBox, kBox, bars + s);
            }
        }
        out[blockIdx.x] = acc;
    }
}

template <int RING>
void run(const uint8_t* src, size_t bytes, int ctas_per_sm, uint32_t* out) {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int smem = RING * 16384 + 1024;
    cudaFuncSetAttribute(k<RING>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int iters = 4000;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float ms = 0;
    for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(e0);
        k<RING><<<sms * ctas_per_sm, 32, smem>>>(src, bytes, iters, out);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
    }
    int clk;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const double tot = double(sms) * ctas_per_sm * iters * 16384.0;
    printf("src %6.1f MB ring %d CTAs/SM %d: %.2f TB/s = %.1f B/clk/SM at %d MHz (%.3f ms, %s)\n", bytes / 1e6, RING,
           ctas_per_sm, tot / (ms * 1e-3) / 1e12, tot / (ms * 1e-3) / (clk * 1e3) / sms, clk / 1000, ms,
           cudaGetErrorString(cudaGetLastError()));
}

int main() {
    uint8_t* src;
    uint32_t* out;
    const size_t big = size_t(1) << 30;
    cudaMalloc(&src, big);
    cudaMemset(src, 1, big);
    cudaMalloc(&out, 4 * 4096);
    for (size_t mb : {32, 64, 1024}) {
        const size_t bytes = mb << 20;
        run<4>(src, bytes, 1, out);
        run<4>(src, bytes, 2, out);
        run<8>(src, bytes, 1, out);
        run<4>(src, bytes, 4, out);
    }
    return 0;
}
