// debug_tile.cu -- a single 128x64 tile through the same tcgen05 / TMEM / TMA building blocks as
// bsa_fwd.cu (S = Q K^T in TMEM, P = bf16(S) back into TMEM, O = P V with an MN-major V operand).
// Used by tests/test_gpu_parity.py::test_debug_tile_mma_layouts to validate the descriptor and
// TMEM-layout conventions in isolation.
#include "internal.h"
#include "ptx.cuh"

namespace pbsa {
namespace {

constexpr uint32_t kTmemCols = 256;

// ---------------------------------------------------------------------- debug tile
// One CTA of 128 threads: q [128][d], k/v [64][d] via TMA; S = q k^T -> s_out; P = bf16(S) -> TMEM;
// O = P v -> o_out.  Same descriptors / TMEM layouts as bsa_fwd_kernel.
template <int D>
__global__ void __launch_bounds__(128, 1)
    debug_tile_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                      const __grid_constant__ CUtensorMap tm_v, float* s_out, float* o_out) {
    constexpr int kHalves = D / 64;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* q_smem = smem;
    uint8_t* k_smem = smem + kHalves * 16384;
    uint8_t* v_smem = k_smem + kHalves * 8192;
    uint64_t* bars = reinterpret_cast<uint64_t*>(v_smem + kHalves * 8192);  // [0] load, [1] mma
    uint32_t* holder = reinterpret_cast<uint32_t*>(bars + 2);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        mbar_init(bars, 1);
        mbar_init(bars + 1, 1);
        fence_barrier_init();
    }
    if (warp == 1) tmem_alloc<kTmemCols>(holder);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *holder;
    if (threadIdx.x == 0) {
        mbar_arrive_expect_tx(bars, kHalves * (16384 + 8192 + 8192));
        for (int h = 0; h < kHalves; ++h) {
            tma_load_2d(q_smem + h * 16384, &tm_q, bars, h * 64, 0);
            tma_load_2d(k_smem + h * 8192, &tm_k, bars, h * 64, 0);
            tma_load_2d(v_smem + h * 8192, &tm_v, bars, h * 64, 0);
        }
        mbar_wait(bars, 0);
        tc_fence_after();
        constexpr uint32_t idesc_s = idesc_bf16_f32(128, 64, 0, 0);
        for (int kk = 0; kk < D / 16; ++kk) {
            const uint32_t off = (kk & 3) * 32;
            mma_ss(tmem + D, smem_desc_sw128(smem_u32(q_smem) + (kk >> 2) * 16384 + off, 16, 1024),
                   smem_desc_sw128(smem_u32(k_smem) + (kk >> 2) * 8192 + off, 16, 1024), idesc_s, kk > 0);
        }
        mma_commit(bars + 1);
    }
    __syncwarp();
    mbar_wait(bars + 1, 0);
    tc_fence_after();
    const int r = warp * 32 + lane;
    const uint32_t t_row = tmem + (static_cast<uint32_t>(warp * 32) << 16);
    uint32_t sr[64];
    tmem_ld32(t_row + D, *reinterpret_cast<uint32_t(*)[32]>(sr));
    tmem_ld32(t_row + D + 32, *reinterpret_cast<uint32_t(*)[32]>(sr + 32));
    tmem_wait_ld();
    for (int c = 0; c < 64; ++c) s_out[r * 64 + c] = __uint_as_float(sr[c]);
    uint32_t pk[32];
    for (int c = 0; c < 32; ++c) pk[c] = pack_bf16x2(__uint_as_float(sr[2 * c]), __uint_as_float(sr[2 * c + 1]));
    tmem_st32(t_row + D, pk);
    tmem_wait_st();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (threadIdx.x == 0) {
        constexpr uint32_t idesc_o = idesc_bf16_f32(128, D, 0, 1);
        for (int kk = 0; kk < 4; ++kk)
            mma_ts(tmem, tmem + D + kk * 8, smem_desc_sw128(smem_u32(v_smem) + kk * 2048, 8192, 1024), idesc_o,
                   kk > 0);
        mma_commit(bars + 1);
    }
    __syncwarp();
    mbar_wait(bars + 1, 1);
    tc_fence_after();
    for (int c0 = 0; c0 < D; c0 += 32) {
        uint32_t ov[32];
        tmem_ld32(t_row + c0, ov);
        tmem_wait_ld();
        for (int c = 0; c < 32; ++c) o_out[r * D + c0 + c] = __uint_as_float(ov[c]);
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc<kTmemCols>(tmem);
    }
}

template <int D>
int launch_debug_impl(const bf16* q, const bf16* k, const bf16* v, float* s_out, float* o_out, cudaStream_t s) {
    alignas(64) CUtensorMap tq, tk, tv;
    std::string err;
    const uint64_t strides[1] = {static_cast<uint64_t>(D) * 2};
    const uint32_t box_q[2] = {64, 128}, box_kv[2] = {64, 64};
    const uint64_t dq[2] = {D, 128}, dkv[2] = {D, 64};
    if (!encode_tmap_bf16(&tq, q, 2, dq, strides, box_q, &err) ||
        !encode_tmap_bf16(&tk, k, 2, dkv, strides, box_kv, &err) ||
        !encode_tmap_bf16(&tv, v, 2, dkv, strides, box_kv, &err))
        return set_error(PBSA_ECUDA, "debug tensor map: " + err);
    const size_t smem = 1024 + (D / 64) * 32768 + 64;
    cudaFuncSetAttribute(debug_tile_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    count_launch();
    debug_tile_kernel<D><<<1, 128, smem, s>>>(tq, tk, tv, s_out, o_out);
    return check_launch("debug_tile_kernel");
}

}  // namespace

int launch_debug_tile(const bf16* q, const bf16* k, const bf16* v, int d, float* s_out, float* o_out,
                      cudaStream_t s) {
    if (d == 128) return launch_debug_impl<128>(q, k, v, s_out, o_out, s);
    return launch_debug_impl<64>(q, k, v, s_out, o_out, s);
}

}  // namespace pbsa
