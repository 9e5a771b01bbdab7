// Probe (perf experiment only): where does a cta_group::1 M=64 tcgen05.mma put its accumulator
// rows in TMEM, which TMEM lanes does an M=64 TS MMA read its A operand from, and what does an
// M=64 MMA cost per K-step next to M=128.  Decides whether K3 can run blocks that only one query
// block of the 128-row tile sees at M=64.
//
// Layout: A[r][0] = r, A[r][1] = 1; B[n][0] = 256, B[n][1] = n  =>  D[r][n] = 256 r + n.  TMEM is
// prefilled with NaN; every lane's 64 columns are dumped and decoded as (source row, column ok).
// For TS the A operand is written into TMEM with lane L holding row L, so the decoded row names
// the lane the operand came from.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <stdint.h>
#include <cuda_bf16.h>
#include "../../paper_2604_21221_b200/csrc/ptx.cuh"
using namespace pbsa;

__device__ __forceinline__ void mma_ws(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                       uint32_t accumulate) {
    asm volatile(
        "{ .reg .pred p; setp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.ws.cta_group::1.kind::f16 [%0], %1, %2, %3, p; }" ::"r"(d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
}

__device__ __forceinline__ uint16_t bf(float x) {
    __nv_bfloat16 h = __float2bfloat16_rn(x);
    return *reinterpret_cast<uint16_t*>(&h);
}

// mode: 0 SS M64 D lane 0 | 1 SS M64 D lane 64 | 2 SS M64 D lane 16 | 3 TS M64 A lane 0 |
//       4 TS M64 A lane 64 | 5 SS M128 | 6 SS M64 with A starting at smem row 64 |
//       7 .ws M64 | 8 .ws M64 D lane 64, A row 64 | 9 .ws M32 | 10 .ws M64 D lane 32
__global__ void layout_kernel(float* out, int mode) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint64_t bar;
    __shared__ uint32_t holder;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint8_t* a_s = smem;            // 128 rows x 128 B (SW128 K-major; only chunk 0 nonzero)
    uint8_t* b_s = smem + 16384;    // 64 rows x 128 B
    for (int i = threadIdx.x; i < 24576 / 16; i += blockDim.x) reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
    __syncthreads();
    {
        const int r = threadIdx.x;  // 128 threads: A rows; first 64 also B rows
        // SW128: 16-byte chunk c of row r lives at chunk position c ^ (r & 7)
        uint16_t* ar = reinterpret_cast<uint16_t*>(a_s + r * 128 + ((0 ^ (r & 7)) * 16));
        ar[0] = bf(static_cast<float>(r));
        ar[1] = bf(1.0f);
        if (r < 64) {
            uint16_t* br = reinterpret_cast<uint16_t*>(b_s + r * 128 + ((0 ^ (r & 7)) * 16));
            br[0] = bf(256.0f);
            br[1] = bf(static_cast<float>(r));
        }
    }
    if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
    if (warp == 0) tmem_alloc<256>(&holder);
    fence_proxy_async_smem();
    tc_fence_before(); __syncthreads(); tc_fence_after();
    const uint32_t tmem = holder;
    const uint32_t t_lane = tmem + (static_cast<uint32_t>(warp * 32) << 16);
    {
        uint32_t v[32];
        for (int c = 0; c < 32; ++c) v[c] = 0x7FC00000u;  // NaN
        tmem_st32(t_lane, v);
        tmem_st32(t_lane + 32, v);
        // TS A operand at column 128: lane L = row L, k0 = L, k1 = 1, rest 0 (8 columns = K16)
        uint32_t a[32];
        for (int c = 0; c < 32; ++c) a[c] = 0;
        a[0] = static_cast<uint32_t>(bf(static_cast<float>(threadIdx.x))) | (static_cast<uint32_t>(bf(1.0f)) << 16);
        tmem_st32(t_lane + 128, a);
        tmem_wait_st();
    }
    tc_fence_before(); __syncthreads(); tc_fence_after();
    if (warp == 0) {
        if (elect_one()) {
            const uint64_t adesc = smem_desc_sw128(smem_u32(a_s), 16, 1024);
            const uint64_t adesc64 = smem_desc_sw128(smem_u32(a_s) + 8192, 16, 1024);
            const uint64_t bdesc = smem_desc_sw128(smem_u32(b_s), 16, 1024);
            const uint32_t i64 = idesc_bf16_f32(64, 64, 0, 0), i128 = idesc_bf16_f32(128, 64, 0, 0);
            switch (mode) {
                case 0: mma_ss(tmem, adesc, bdesc, i64, 0); break;
                case 1: mma_ss(tmem + (64u << 16), adesc, bdesc, i64, 0); break;
                case 2: mma_ss(tmem + (16u << 16), adesc, bdesc, i64, 0); break;
                case 3: mma_ts(tmem, tmem + 128, bdesc, i64, 0); break;
                case 4: mma_ts(tmem, tmem + (64u << 16) + 128, bdesc, i64, 0); break;
                case 5: mma_ss(tmem, adesc, bdesc, i128, 0); break;
                case 6: mma_ss(tmem, adesc64, bdesc, i64, 0); break;
                case 7: mma_ws(tmem, adesc, bdesc, i64, 0); break;
                case 8: mma_ws(tmem + (64u << 16), adesc64, bdesc, i64, 0); break;
                case 9: mma_ws(tmem, adesc, bdesc, idesc_bf16_f32(32, 64, 0, 0), 0); break;
                case 10: mma_ws(tmem + (32u << 16), adesc, bdesc, i64, 0); break;
            }
            mma_commit(&bar);
        }
        __syncwarp();
    }
    mbar_wait(&bar, 0);
    tc_fence_after();
    uint32_t v[64];
    tmem_ld32(t_lane, *reinterpret_cast<uint32_t(*)[32]>(v));
    tmem_ld32(t_lane + 32, *reinterpret_cast<uint32_t(*)[32]>(v + 32));
    tmem_wait_ld();
    for (int c = 0; c < 64; ++c) out[threadIdx.x * 64 + c] = __uint_as_float(v[c]);
    tc_fence_before(); __syncthreads();
    if (warp == 0) { tc_fence_after(); tmem_dealloc<256>(tmem); }
}

// Throughput: one elected thread issues iters x 8 MMAs back to back.
template <int M, int N, int TS>
__global__ void tput_kernel(long long* out, int iters) {
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
        constexpr uint32_t idesc = idesc_bf16_f32(M, N, 0, 0);
        long long t0 = clock64();
        if (elect_one()) {
            for (int it = 0; it < iters; ++it) {
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) {
                    if (TS == 2) mma_ws(tmem + 256, adesc + (((kk & 3) * 32) >> 4), bdesc + (((kk & 3) * 32) >> 4), idesc, 1u);
                    else if (TS) mma_ts(tmem + 256, tmem + 448 + kk * 8 % 64, bdesc + (((kk & 3) * 32) >> 4), idesc, 1u);
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

template <int M, int N, int TS>
void tput(const char* name) {
    long long* out; cudaMalloc(&out, 148 * 8);
    const int iters = 2000;
    cudaFuncSetAttribute(tput_kernel<M, N, TS>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
    tput_kernel<M, N, TS><<<148, 128, 65536>>>(out, iters);
    tput_kernel<M, N, TS><<<148, 128, 65536>>>(out, iters);
    cudaDeviceSynchronize();
    long long h[148]; cudaMemcpy(h, out, sizeof(h), cudaMemcpyDeviceToHost);
    double avg = 0; for (int i = 0; i < 148; ++i) avg += h[i]; avg /= 148;
    printf("%-4s M=%3d N=%3d K16: %.1f cycles per MMA  err=%s\n", name, M, N, avg / (iters * 8.0),
           cudaGetErrorString(cudaGetLastError()));
    cudaFree(out);
}

int main(int argc, char** argv) {
    if (argc > 1 && !strcmp(argv[1], "tput")) {
        tput<128, 64, 0>("SS");
        tput<64, 64, 0>("SS");
        tput<128, 128, 0>("SS");
        tput<64, 128, 0>("SS");
        tput<128, 128, 1>("TS");
        tput<64, 128, 1>("TS");
        tput<64, 64, 1>("TS");
        tput<64, 64, 2>("WS");
        tput<128, 64, 2>("WS");
        tput<32, 64, 2>("WS");
        tput<64, 128, 2>("WS");
        return 0;
    }
    const int mode = argc > 1 ? atoi(argv[1]) : 0;
    float* d; cudaMalloc(&d, 128 * 64 * 4);
    cudaFuncSetAttribute(layout_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768);
    layout_kernel<<<1, 128, 32768>>>(d, mode);
    cudaError_t e = cudaDeviceSynchronize();
    printf("mode %d: %s\n", mode, cudaGetErrorString(e));
    if (e != cudaSuccess) return 1;
    static float h[128 * 64];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    // per lane: "." untouched, "r" = source row (all 64 columns consistent), "?" = mixed
    for (int L = 0; L < 128; ++L) {
        int nan = 0, row = -1, ok = 1;
        for (int c = 0; c < 64; ++c) {
            const float x = h[L * 64 + c];
            if (std::isnan(x)) { ++nan; continue; }
            const int r = static_cast<int>(x) / 256, n = static_cast<int>(x) % 256;
            if (row < 0) row = r;
            if (r != row || n != c) ok = 0;
        }
        if (nan == 64) printf("  L%3d: .\n", L);
        else if (nan == 0 && ok) printf("  L%3d: row %d\n", L, row);
        else {
            printf("  L%3d: mixed nan=%d:", L, nan);
            for (int c = 0; c < 8; ++c) printf(" %g", h[L * 64 + c]);
            printf("\n");
        }
    }
    return 0;
}
