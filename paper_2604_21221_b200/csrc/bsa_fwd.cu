// bsa_fwd.cu -- K3 block-sparse attention forward on tcgen05 / TMEM / TMA (sm_100a).
//
// Reference op: attention.attention_sparse: for each query block, softmax over
// the persistent blocks + current chunk (dense, Eq. 5) and the Top-K selected
// local blocks (Eq. 11), online softmax, masked blocks never loaded.
//
// Work unit: one CTA = one 128-row query tile = two consecutive query blocks (rows [0,64) hold
// query block 2t, rows [64,128) block 2t+1; rows >= b of each half are padding).  The CTA walks
// the UNION of both blocks' visible key blocks; a 2-bit mask per list entry tells each half
// whether the key block is visible to it (invisible -> probabilities forced to 0).  Dense blocks
// are visible to both halves, so only the selected local blocks cost union overhead.  (M=128 is
// the full-rate tcgen05 shape; an M=64 tile per query block would run at half rate.)
//
// Warp roles (192 threads):
//   warp 0  TMA producer: Q (3-D map over [unit*nqb][b][d], box b rows -> 64-row half),
//           K and V slots (2-D map over the slot pools, one 64x64 box per d-half)
//   warp 1  tcgen05 issuer: S_j = Q K_j^T (SS, M=128 N=64, fp32 in TMEM), O += P_j V_j
//           (TS: P in TMEM as bf16, V MN-major from smem), commits to mbarriers
//   warps 2-5  softmax: thread = query row = TMEM lane; online softmax with lazy rescale
//           (only when the running max grows by > 8 in log2 units), P written back into the
//           S columns as packed bf16, final O / l epilogue straight from TMEM to HBM.
// TMEM: O [0, d), S0 [d, d+64), S1 [d+64, d+128) -> 256 columns, so two CTAs fit per SM.
//
// Roofline: tensor core.  Executed FLOPs per tile = 4 * 128 * 64 * d * |union list|.
#include <cfloat>
#include <cstdlib>

#include "internal.h"
#include "ptx.cuh"

namespace pbsa {
namespace {

constexpr int kThreads = 192;
constexpr uint32_t kTmemCols = 256;
constexpr float kRescaleThreshold = 8.0f;  // log2 units

struct BsaParams {
    int units, nqb, b, n_slots;
    const int32_t* dense;
    int dense_stride, n_dense;
    const int32_t* local;
    int local_stride, n_local;
    const int32_t* sel;
    int k;
    bf16* o;
    float* lse;
    float scale_log2;
    int max_list, bm_words;
    int ablate;  // perf experiments only (PBSA_ABLATE): 1 = softmax writes P=0 without computing
};

template <int D, int NSK, int NSV>
struct Layout {
    static constexpr int kHalves = D / 64;
    static constexpr uint32_t kQBytes = kHalves * 128 * 128;  // [half][128 rows][128 B]
    static constexpr uint32_t kKVBytes = kHalves * 64 * 128;  // one slot: [half][64 rows][128 B]
    static constexpr uint32_t kOffQ = 0;
    static constexpr uint32_t kOffK = kOffQ + kQBytes;
    static constexpr uint32_t kOffV = kOffK + NSK * kKVBytes;
    static constexpr uint32_t kOffBar = kOffV + NSV * kKVBytes;
    static constexpr int kNumBars = 1 + 2 * NSK + 2 * NSV + 6;
    static constexpr uint32_t kOffMisc = kOffBar + kNumBars * 8;
    static constexpr uint32_t kOffList = kOffMisc + 16;
    static constexpr uint32_t kSColBase = D;  // S0 at D, S1 at D + 64
    static size_t bytes(int max_list, int bm_words) {
        return 1024 + kOffList + static_cast<size_t>(max_list) * 4 + static_cast<size_t>(bm_words) * 8;
    }
};

template <int D, int NSK, int NSV, int B>
__global__ void __launch_bounds__(kThreads, 2)
    bsa_fwd_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                   const __grid_constant__ CUtensorMap tm_v, const BsaParams p) {
    using L = Layout<D, NSK, NSV>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* q_smem = smem + L::kOffQ;
    uint8_t* k_smem = smem + L::kOffK;
    uint8_t* v_smem = smem + L::kOffV;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::kOffBar);
    uint64_t* q_full = bars;
    uint64_t* k_full = bars + 1;
    uint64_t* k_empty = k_full + NSK;
    uint64_t* v_full = k_empty + NSK;
    uint64_t* v_empty = v_full + NSV;
    uint64_t* s_full = v_empty + NSV;
    uint64_t* p_full = s_full + 2;
    uint64_t* o_done = p_full + 2;
    uint32_t* misc = reinterpret_cast<uint32_t*>(smem + L::kOffMisc);  // [0] tmem base, [1] list len
    int32_t* list = reinterpret_cast<int32_t*>(smem + L::kOffList);
    uint32_t* bm = reinterpret_cast<uint32_t*>(list + p.max_list);  // [2][bm_words]

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int tile = blockIdx.x, u = blockIdx.y;
    const int qb0 = 2 * tile;
    const bool has2 = qb0 + 1 < p.nqb;

    // ------------------------------------------------------------------ setup
    if (warp == 0 && lane == 0) {
        mbar_init(q_full, 1);
        for (int s = 0; s < NSK; ++s) {
            mbar_init(k_full + s, 1);
            mbar_init(k_empty + s, 1);
        }
        for (int s = 0; s < NSV; ++s) {
            mbar_init(v_full + s, 1);
            mbar_init(v_empty + s, 1);
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init(s_full + s, 1);
            mbar_init(p_full + s, 128);
            mbar_init(o_done + s, 1);
        }
        fence_barrier_init();
        tma_prefetch(&tm_q);
        tma_prefetch(&tm_k);
        tma_prefetch(&tm_v);
    }
    if (warp == 1) tmem_alloc<kTmemCols>(misc);
    if (warp >= 2) {
        // visible-list construction: dense blocks (both halves) ++ union of the two selections
        const int t = threadIdx.x - 64;
        const int sel_rows = has2 ? 2 : 1;
        for (int w = t; w < 2 * p.bm_words; w += 128) bm[w] = 0u;
        // zero the query padding rows (rows >= b of each half, the whole upper half without a
        // second query block) so their S rows stay finite; TMA only writes rows < b
        {
            const int pad = 64 - p.b;
            const int rows_pad = has2 ? 2 * pad : pad + 64;
            for (int e = t; e < rows_pad * L::kHalves * 8; e += 128) {
                const int chunk = e & 7, rh = e >> 3;
                const int h = rh % L::kHalves, pr = rh / L::kHalves;
                const int row = pr < pad ? p.b + pr : (has2 ? 64 + p.b + (pr - pad) : 64 + (pr - pad));
                *reinterpret_cast<uint4*>(q_smem + h * 16384 + row * 128 + chunk * 16) = make_uint4(0, 0, 0, 0);
            }
            fence_proxy_async_smem();
        }
        named_bar_sync(1, 128);
        if (p.k > 0 && p.n_local > 0) {
            for (int e = t; e < sel_rows * p.k; e += 128) {
                const int r = e / p.k, c = e % p.k;
                const int idx = __ldg(p.sel + (static_cast<int64_t>(u) * p.nqb + qb0 + r) * p.k + c);
                atomicOr(&bm[r * p.bm_words + (idx >> 5)], 1u << (idx & 31));
            }
        }
        for (int e = t; e < p.n_dense; e += 128)
            list[e] = __ldg(p.dense + static_cast<int64_t>(u) * p.dense_stride + e) | (3 << 24);
        named_bar_sync(1, 128);
        if (warp == 2) {
            int run = p.n_dense;
            const int32_t* loc = p.local + static_cast<int64_t>(u) * p.local_stride;
            for (int w0 = 0; w0 < p.bm_words; w0 += 32) {
                const int w = w0 + lane;
                const uint32_t a = w < p.bm_words ? bm[w] : 0u;
                const uint32_t c = w < p.bm_words ? bm[p.bm_words + w] : 0u;
                uint32_t un = a | c;
                const int cnt = __popc(un);
                int incl = cnt;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int y = __shfl_up_sync(0xffffffffu, incl, o);
                    if (lane >= o) incl += y;
                }
                int pos = run + incl - cnt;
                while (un) {
                    const int bit = __ffs(un) - 1;
                    un &= un - 1;
                    const int idx = w * 32 + bit;
                    const int mask = static_cast<int>((a >> bit) & 1u) | (static_cast<int>((c >> bit) & 1u) << 1);
                    list[pos++] = __ldg(loc + idx) | (mask << 24);
                }
                run += __shfl_sync(0xffffffffu, incl, 31);
            }
            if (lane == 0) misc[1] = static_cast<uint32_t>(run);
        }
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = misc[0];
    const int n = static_cast<int>(misc[1]);

    if (warp == 0) {
        // ============================================================== TMA producer
        if (lane == 0) {
            const uint32_t qbytes = (has2 ? 2u : 1u) * L::kHalves * static_cast<uint32_t>(p.b) * 128u;
            mbar_arrive_expect_tx(q_full, qbytes);
            for (int r = 0; r < (has2 ? 2 : 1); ++r)
                for (int h = 0; h < L::kHalves; ++h)
                    tma_load_3d(q_smem + h * 16384 + r * 8192, &tm_q, q_full, h * 64, 0,
                                u * p.nqb + qb0 + r);
            auto load_v = [&](int j) {
                const int s = j % NSV;
                mbar_wait(v_empty + s, ((j / NSV) & 1) ^ 1);
                mbar_arrive_expect_tx(v_full + s, L::kKVBytes);
                const int row0 = (u * p.n_slots + (list[j] & 0xFFFFFF)) * 64;
                for (int h = 0; h < L::kHalves; ++h)
                    tma_load_2d(v_smem + s * L::kKVBytes + h * 8192, &tm_v, v_full + s, h * 64, row0);
            };
            for (int j = 0; j < n; ++j) {
                const int s = j % NSK;
                mbar_wait(k_empty + s, ((j / NSK) & 1) ^ 1);
                mbar_arrive_expect_tx(k_full + s, L::kKVBytes);
                const int row0 = (u * p.n_slots + (list[j] & 0xFFFFFF)) * 64;
                for (int h = 0; h < L::kHalves; ++h)
                    tma_load_2d(k_smem + s * L::kKVBytes + h * 8192, &tm_k, k_full + s, h * 64, row0);
                if (j >= 1) load_v(j - 1);
            }
            if (n > 0) load_v(n - 1);
        }
    } else if (warp == 1) {
        // ============================================================== tcgen05 issuer
        if (lane == 0 && n > 0) {
            constexpr uint32_t idesc_s = idesc_bf16_f32(128, 64, 0, 0);
            constexpr uint32_t idesc_o = idesc_bf16_f32(128, D, 0, 1);
            const uint32_t q_base = smem_u32(q_smem);
            const uint32_t k_base = smem_u32(k_smem);
            const uint32_t v_base = smem_u32(v_smem);
            mbar_wait(q_full, 0);
            tc_fence_after();
            auto issue_s = [&](int j) {
                const int s = j % NSK;
                mbar_wait(k_full + s, (j / NSK) & 1);
                tc_fence_after();
                const uint32_t d_tmem = tmem + L::kSColBase + (j & 1) * 64;
#pragma unroll
                for (int kk = 0; kk < D / 16; ++kk) {
                    const uint32_t off = (kk & 3) * 32;
                    const uint64_t a = smem_desc_sw128(q_base + (kk >> 2) * 16384 + off, 16, 1024);
                    const uint64_t b = smem_desc_sw128(k_base + s * L::kKVBytes + (kk >> 2) * 8192 + off, 16, 1024);
                    mma_ss(d_tmem, a, b, idesc_s, kk > 0 ? 1u : 0u);
                }
                mma_commit(k_empty + s);
                mma_commit(s_full + (j & 1));
            };
            issue_s(0);
            for (int j = 0; j < n; ++j) {
                if (j + 1 < n) issue_s(j + 1);
                const int sv = j % NSV;
                mbar_wait(p_full + (j & 1), (j >> 1) & 1);
                mbar_wait(v_full + sv, (j / NSV) & 1);
                tc_fence_after();
                const uint32_t a_tmem = tmem + L::kSColBase + (j & 1) * 64;
#pragma unroll
                for (int kk = 0; kk < 4; ++kk) {
                    const uint64_t b = smem_desc_sw128(v_base + sv * L::kKVBytes + kk * 2048, 8192, 1024);
                    mma_ts(tmem, a_tmem + kk * 8, b, idesc_o, (j > 0 || kk > 0) ? 1u : 0u);
                }
                mma_commit(v_empty + sv);
                mma_commit(o_done + (j & 1));
            }
        }
    } else {
        // ============================================================== softmax warps
        const int quarter = warp & 3;
        const int r = quarter * 32 + lane;
        const int half = r >> 6, rr = r & 63;
        const int qb = qb0 + half;
        const bool valid = rr < p.b && qb < p.nqb;
        const uint32_t lane_base = static_cast<uint32_t>(quarter * 32) << 16;
        const uint32_t t_o = tmem + lane_base;
        float m = -INFINITY, l = 0.0f;
        int o_waited[2] = {0, 0};
        auto pv_done = [&](int x) {  // wait until PV_x has completed
            if (x < 0) return;
            const int bb = x & 1;
            const int need = (x >> 1) + 1;
            while (o_waited[bb] < need) {
                mbar_wait(o_done + bb, o_waited[bb] & 1);
                ++o_waited[bb];
            }
        };
        // columns >= BB of a slot are padding (compile-time for the common block sizes)
        constexpr int BB = B > 0 ? B : 64;
        const int bcols = B > 0 ? B : p.b;
        const float2 scl2 = make_float2(p.scale_log2, p.scale_log2);
        for (int j = 0; j < n; ++j) {
            const int buf = j & 1;
            mbar_wait(s_full + buf, (j >> 1) & 1);
            tc_fence_after();
            pv_done(j - 2);  // already complete: S_j was committed after PV_{j-2}
            const uint32_t t_s = t_o + L::kSColBase + buf * 64;
            uint32_t pk[32];
            // rows of one warp all lie in one half -> visibility is warp-uniform
            const bool vis = ((list[j] >> (24 + half)) & 1) && p.ablate != 1;
            if (vis) {
                uint32_t sr[64];
                tmem_ld32(t_s, *reinterpret_cast<uint32_t(*)[32]>(sr));
                tmem_ld32(t_s + 32, *reinterpret_cast<uint32_t(*)[32]>(sr + 32));
                tmem_wait_ld();
                float sv[64];
#pragma unroll
                for (int c = 0; c < 64; ++c) {
                    sv[c] = __uint_as_float(sr[c]);
                    if (B == 0 && c >= bcols) sv[c] = -INFINITY;  // generic block size
                }
                // row max over the valid columns: FMNMX3 tree
                float mx4[4];
#pragma unroll
                for (int t = 0; t < 4; ++t) {
                    float a = -INFINITY;
#pragma unroll
                    for (int c = t * 16; c < t * 16 + 16; c += 2) {
                        if (c + 1 < BB) a = fmax3(a, sv[c], sv[c + 1]);
                        else if (c < BB) a = fmaxf(a, sv[c]);
                    }
                    mx4[t] = a;
                }
                float mx = fmaxf(fmaxf(mx4[0], mx4[1]), fmaxf(mx4[2], mx4[3])) * p.scale_log2;
                if (!valid) mx = -INFINITY;
                float factor = 1.0f;
                bool resc = false;
                if (mx > m) {
                    if (m == -INFINITY) {
                        m = mx;  // first visible block for this row: its O row is still zero
                    } else if (mx > m + kRescaleThreshold) {
                        factor = exp2_approx(m - mx);
                        m = mx;
                        resc = true;
                    }
                }
                if (__any_sync(0xffffffffu, resc)) {
                    pv_done(j - 1);
                    tc_fence_after();
#pragma unroll 1
                    for (int c0 = 0; c0 < D; c0 += 32) {
                        uint32_t ov[32];
                        tmem_ld32(t_o + c0, ov);
                        tmem_wait_ld();
#pragma unroll
                        for (int c = 0; c < 32; ++c) ov[c] = __float_as_uint(__uint_as_float(ov[c]) * factor);
                        tmem_st32(t_o + c0, ov);
                    }
                    l *= factor;
                }
                // p = 2^(s*scale_log2 - m); padding rows get bias -inf -> p = 0
                const float bias = valid ? -m : -INFINITY;
                const float2 bias2 = make_float2(bias, bias);
                float2 acc[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f),
                                 make_float2(0.f, 0.f)};
#pragma unroll
                for (int c2 = 0; c2 < 32; ++c2) {
                    const float2 x = __ffma2_rn(make_float2(sv[2 * c2], sv[2 * c2 + 1]), scl2, bias2);
                    float2 e;
                    e.x = (2 * c2 < BB) ? exp2_approx(x.x) : 0.0f;
                    e.y = (2 * c2 + 1 < BB) ? exp2_approx(x.y) : 0.0f;
                    if (B == 0) {
                        if (2 * c2 >= bcols) e.x = 0.0f;
                        if (2 * c2 + 1 >= bcols) e.y = 0.0f;
                    }
                    acc[c2 & 3] = __fadd2_rn(acc[c2 & 3], e);
                    pk[c2] = pack_bf16x2(e.x, e.y);
                }
                const float2 s01 = __fadd2_rn(__fadd2_rn(acc[0], acc[1]), __fadd2_rn(acc[2], acc[3]));
                l += s01.x + s01.y;
            } else {
#pragma unroll
                for (int c = 0; c < 32; ++c) pk[c] = 0u;
            }
            tmem_st32(t_s, pk);
            tmem_wait_st();
            tc_fence_before();
            mbar_arrive(p_full + buf);
        }
        pv_done(n - 2);
        pv_done(n - 1);
        tc_fence_after();
        // epilogue: O / l -> bf16 -> HBM
        const float inv = l > 0.0f ? 1.0f / l : 0.0f;
        bf16* orow = p.o + ((static_cast<int64_t>(u) * p.nqb + qb) * p.b + rr) * D;
#pragma unroll 1
        for (int c0 = 0; c0 < D; c0 += 32) {
            uint32_t ov[32];
            if (n > 0) {
                tmem_ld32(t_o + c0, ov);
                tmem_wait_ld();
            } else {
#pragma unroll
                for (int c = 0; c < 32; ++c) ov[c] = 0u;
            }
            if (valid) {
                uint4 pkd[4];
                uint32_t* w = reinterpret_cast<uint32_t*>(pkd);
#pragma unroll
                for (int c = 0; c < 16; ++c)
                    w[c] = pack_bf16x2(__uint_as_float(ov[2 * c]) * inv, __uint_as_float(ov[2 * c + 1]) * inv);
                uint4* dst = reinterpret_cast<uint4*>(orow + c0);
#pragma unroll
                for (int c = 0; c < 4; ++c) dst[c] = pkd[c];
            }
        }
        if (valid && p.lse != nullptr)
            p.lse[(static_cast<int64_t>(u) * p.nqb + qb) * p.b + rr] =
                l > 0.0f ? (m + __log2f(l)) * 0.69314718055994531f : -INFINITY;
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc<kTmemCols>(tmem);
    }
}

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

template <int D, int NSK, int NSV, int B>
int launch_impl(const bf16* q, const bf16* kp, const bf16* vp, const BsaParams& p, cudaStream_t s) {
    using L = Layout<D, NSK, NSV>;
    alignas(64) CUtensorMap tq, tk, tv;
    std::string err;
    {
        const uint64_t dims[3] = {static_cast<uint64_t>(D), static_cast<uint64_t>(p.b),
                                  static_cast<uint64_t>(p.units) * p.nqb};
        const uint64_t strides[2] = {static_cast<uint64_t>(D) * 2, static_cast<uint64_t>(p.b) * D * 2};
        const uint32_t box[3] = {64, static_cast<uint32_t>(p.b), 1};
        if (!encode_tmap_bf16(&tq, q, 3, dims, strides, box, &err))
            return set_error(PBSA_ECUDA, "tensor map Q: " + err);
    }
    {
        const uint64_t dims[2] = {static_cast<uint64_t>(D), static_cast<uint64_t>(p.units) * p.n_slots * 64};
        const uint64_t strides[1] = {static_cast<uint64_t>(D) * 2};
        const uint32_t box[2] = {64, 64};
        if (!encode_tmap_bf16(&tk, kp, 2, dims, strides, box, &err))
            return set_error(PBSA_ECUDA, "tensor map K: " + err);
        if (!encode_tmap_bf16(&tv, vp, 2, dims, strides, box, &err))
            return set_error(PBSA_ECUDA, "tensor map V: " + err);
    }
    const size_t smem = L::bytes(p.max_list, p.bm_words);
    if (smem > 227 * 1024)
        return set_error(PBSA_EUNSUPPORTED, "bsa_fwd: visible list too long for shared memory");
    static bool configured = false;
    if (!configured) {
        cudaFuncSetAttribute(bsa_fwd_kernel<D, NSK, NSV, B>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
        configured = true;
    }
    dim3 grid((p.nqb + 1) / 2, p.units);
    bsa_fwd_kernel<D, NSK, NSV, B><<<grid, kThreads, smem, s>>>(tq, tk, tv, p);
    return check_launch("bsa_fwd_kernel");
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
    debug_tile_kernel<D><<<1, 128, smem, s>>>(tq, tk, tv, s_out, o_out);
    return check_launch("debug_tile_kernel");
}

}  // namespace

int launch_bsa_fwd(const bf16* q, const bf16* k_pool, const bf16* v_pool, int n_slots,
                   const int32_t* dense, int dense_stride, int n_dense, const int32_t* local,
                   int local_stride, int n_local, const int32_t* sel, int k, int nqb, int b, int d,
                   int units, float scale, bf16* o, float* lse, cudaStream_t s) {
    BsaParams p{};
    p.units = units;
    p.nqb = nqb;
    p.b = b;
    p.n_slots = n_slots;
    p.dense = dense;
    p.dense_stride = dense_stride;
    p.n_dense = n_dense;
    p.local = local;
    p.local_stride = local_stride;
    p.n_local = n_local;
    p.sel = sel;
    p.k = (n_local > 0) ? k : 0;
    p.o = o;
    p.lse = lse;
    p.scale_log2 = scale * 1.4426950408889634f;
    {
        static const int ablate = getenv("PBSA_ABLATE") ? atoi(getenv("PBSA_ABLATE")) : 0;
        p.ablate = ablate;
    }
    p.bm_words = (n_local + 31) / 32 + 1;
    p.max_list = n_dense + (p.k > 0 ? (2 * p.k < n_local ? 2 * p.k : n_local) : 0);
    if (units == 0 || nqb == 0) return 0;
    if (d == 128) {
        if (b == 60) return launch_impl<128, 2, 2, 60>(q, k_pool, v_pool, p, s);
        if (b == 64) return launch_impl<128, 2, 2, 64>(q, k_pool, v_pool, p, s);
        return launch_impl<128, 2, 2, 0>(q, k_pool, v_pool, p, s);
    }
    if (b == 60) return launch_impl<64, 3, 3, 60>(q, k_pool, v_pool, p, s);
    if (b == 64) return launch_impl<64, 3, 3, 64>(q, k_pool, v_pool, p, s);
    return launch_impl<64, 3, 3, 0>(q, k_pool, v_pool, p, s);
}

int launch_debug_tile(const bf16* q, const bf16* k, const bf16* v, int d, float* s_out, float* o_out,
                      cudaStream_t s) {
    if (d == 128) return launch_debug_impl<128>(q, k, v, s_out, o_out, s);
    return launch_debug_impl<64>(q, k, v, s_out, o_out, s);
}

}  // namespace pbsa
