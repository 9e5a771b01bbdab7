// bsa_bwd.cu -- PBSA backward (the paper's training path, Alg. 2,
// PAPER.md:587-626, bwd latencies PAPER.md:845-897).  The reference ships no backward; the
// oracle is the derivative of attention_sparse (oracle/pbsa_oracle.cpp, pinned to torch autograd).
//
// With P = softmax(s * scale) over a row's visible tokens (P = exp(s * scale - lse), lse from the
// forward), dP = dO V^T, D = rowsum(dO o O), dS = P o (dP - D):
//   dQ = scale * dS K        (query-tile-centric kernel: the forward's tile walk + one more MMA)
//   dV = P^T dO, dK = scale * dS^T Q   (KV-centric kernel: a pair of key blocks is the 128-row
//                            tile and the query blocks that see either block are the "keys")
// Every MMA has one of the forward's two shapes: M128 N64 K=d (SS, both operands K-major) or
// M128 N=d K64 (A = bf16 P/dS from TMEM, B = a 64-row block as an MN-major operand).  No online
// softmax is needed -- lse is known -- so each block is one exp2 per element.
//
// Kernels (1 CTA per SM: TMEM holds an accumulator plus double-buffered score tiles):
//   bwd_rows_kernel   D = rowsum(dO o O), lse * log2(e) into a padded workspace
//   bwd_inv_kernel    per local block, the bitmap of query blocks that selected it (from sel)
//   bwd_dq_kernel     warp 0 list + TMA (Q, dO per tile; K, V per block), warp 1 tcgen05
//                     (S = Q K^T, dP = dO V^T, dQ += dS K), warps 2-5 dS (thread = query row)
//   bwd_dkdv_kernel   warp 0 list + TMA (K, V pair per item; Q, dO, lse, D per query block),
//                     warp 1 tcgen05 (S^T = K Q^T, dP^T = V dO^T, dV += P^T dO, dK += dS^T Q),
//                     warps 2-5 P^T and dS^T (thread = key row)
#include <cfloat>
#include <cstdlib>

#include "internal.h"
#include "ptx.cuh"

namespace pbsa {
namespace {

// B-operand ring depth: a stage is held from its TMA load until the block's LAST MMA (dQ, or dV/dK)
// completes -- two blocks of work later -- so two stages left the MMA warp waiting on TMA latency
// every block; four keep the loads a full block ahead.
constexpr int kNS = 4;
// dQ kernel TMEM: dQ [0, 128), Q [128, 192) and dO [192, 256) as bf16 pairs (the A operands of
// S = Q K^T and dP = dO V^T are TMEM-resident: TS MMAs run at the N = 64 floor, SS ones do not),
// then kSB buffers of S (64 columns) + dP (64 columns)
constexpr int kSB = 2;
constexpr uint32_t kQCol = 128, kDOCol = 192, kBufCol = 256;
constexpr int kBwdThreads = 320;  // warp 0 producer, warp 1 MMA, warps 2-9 elementwise
constexpr int kEw = 8;             // elementwise warps: warp w reads TMEM lane quarter w % 4 and
                                   // column half (w - 2) / 4 -- every element is independent (lse is
                                   // known, no row reduction), so the halves never synchronise
constexpr uint32_t kBwdTmemCols = 512;

struct BwdParams {
    int units, nqb, b, n_slots;
    const int32_t* dense;
    int dense_stride, n_dense;
    const int32_t* local;
    int local_stride, n_local;
    const int32_t* sel;
    int k;
    float scale, scale_log2;
    const float* lse2;   // [units * nqb][64] lse * log2(e) (+inf for rows without visible keys)
    const float* drow;   // [units * nqb][64] rowsum(dO o O); rows >= b zero (64-row staging copies)
    const uint32_t* inv;  // [units][n_local][inv_words] query blocks selecting each local block
    int inv_words;
    const bf16* q;       // [units][n_q][d] (dQ kernel: rows go straight to TMEM)
    const bf16* d_o;
    float* dq;           // [units][n_q][d] f32
    float* dk;           // [units][n_slots][64][d] f32
    float* dv;
    int max_list, bm_words, tiles_per_unit, n_tiles;
    int dense_pairs, local_pairs, n_items;
    long long* trace;    // handshake timeline (CTA 0), compiled in only with -DPBSA_K3_TRACE
};

__device__ __forceinline__ void bstamp(const BwdParams& p, int ev, int j) {
#ifdef PBSA_K3_TRACE
    if (p.trace != nullptr && blockIdx.x == 0 && j < 256) p.trace[ev * 256 + j] = clock64();
#else
    (void)p; (void)ev; (void)j;
#endif
}

// ---------------------------------------------------------------------------------- prep
__global__ void bwd_rows_kernel(const bf16* __restrict__ o, const bf16* __restrict__ d_o, const float* __restrict__ lse,
                                int64_t rows, int d, int b, float* __restrict__ lse2, float* __restrict__ drow) {
    pdl_wait();
    const int64_t r = static_cast<int64_t>(blockIdx.x) * (blockDim.x / 32) + threadIdx.x / 32;
    const int lane = threadIdx.x & 31;
    if (r >= rows) return;
    float acc = 0.0f;
    for (int c = lane * 2; c < d; c += 64) {
        const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(o + r * d + c));
        const float2 g = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(d_o + r * d + c));
        acc = fmaf(a.x, g.x, fmaf(a.y, g.y, acc));
    }
#pragma unroll
    for (int s = 16; s; s >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, s);
    if (lane == 0) {
        const int64_t pr = (r / b) * 64 + r % b;  // 64 floats per query block: 256-byte aligned rows
        drow[pr] = acc;
        const float l = lse[r];
        lse2[pr] = l == -INFINITY ? INFINITY : l * 1.4426950408889634f;
    }
}

__global__ void bwd_inv_kernel(const int32_t* __restrict__ sel, int units, int nqb, int k, int n_local, int words,
                               uint32_t* __restrict__ inv) {
    pdl_wait();
    const int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (e >= static_cast<int64_t>(units) * nqb * k) return;
    const int u = static_cast<int>(e / (static_cast<int64_t>(nqb) * k));
    const int i = static_cast<int>((e / k) % nqb);
    const int l = __ldg(sel + e);
    atomicOr(inv + (static_cast<int64_t>(u) * n_local + l) * words + (i >> 5), 1u << (i & 31));
}

// TMEM column of the packed bf16 K16 step kk of a 64-key P / dS tile: the elementwise warp of column
// half h writes its 16 packed columns at [32 h, 32 h + 16) -- inside the fp32 columns it read
__device__ __forceinline__ uint32_t kA(int kk) { return kk < 2 ? kk * 8 : 32 + (kk - 2) * 8; }

// shared-memory layout of both tcgen05 kernels: A tile (128 rows) x2, B stages, barriers, list
template <int D>
struct BwdLayout {
    static constexpr int kHalves = D / 64;
    static constexpr uint32_t kTile = kHalves * 128 * 128;  // 128 rows x D bf16, [half][row][128 B]
    static constexpr uint32_t kBlk = kHalves * 64 * 128;    // 64 rows x D bf16
    // dq:   A0 = Q tile, A1 = dO tile, B stages = K x2, V x2
    // dkdv: A0 = K pair, A1 = V pair, B stages = Q x2, dO x2 (+ lse/D rows per stage)
    static constexpr uint32_t kOffA0 = 0;
    static constexpr uint32_t kOffA1 = kOffA0 + kTile;
    static constexpr uint32_t kOffB = kOffA1 + kTile;  // [2 operands][kNS stages] x kBlk
    static constexpr uint32_t kOffRow = kOffB + 2 * kNS * kBlk;  // [kNS stages][2][64] f32 (dkdv: lse2, D)
    static constexpr uint32_t kOffBar = kOffRow + kNS * 2 * 64 * 4;
    static constexpr int kNumBars = 32;
    static constexpr uint32_t kOffMeta = kOffBar + kNumBars * 8;  // [2][4] ints
    static constexpr uint32_t kOffMisc = kOffMeta + 2 * 4 * 4;
    static constexpr uint32_t kOffList = kOffMisc + 16;
    static size_t bytes(int max_list, int bm_words) {
        return 1024 + kOffList + 2 * static_cast<size_t>(max_list) * 4 + 2 * static_cast<size_t>(bm_words) * 4;
    }
};

// ---------------------------------------------------------------------------------- dQ
template <int D>
__global__ void __launch_bounds__(kBwdThreads, 1)
    bwd_dq_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_do,
                  const __grid_constant__ CUtensorMap tm_k, const __grid_constant__ CUtensorMap tm_v,
                  const BwdParams p) {
    using L = BwdLayout<D>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* q_s = smem + L::kOffA0;
    uint8_t* do_s = smem + L::kOffA1;
    uint8_t* k_s = smem + L::kOffB;                  // [kNS] stages
    uint8_t* v_s = smem + L::kOffB + kNS * L::kBlk;  // [kNS] stages
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::kOffBar);
    uint64_t* q_full = bars + 0;
    uint64_t* q_empty = bars + 1;
    uint64_t* k_full = bars + 2;             // [kNS]
    uint64_t* k_empty = k_full + kNS;        // [kNS]
    uint64_t* v_full = k_empty + kNS;        // [kNS]
    uint64_t* v_empty = v_full + kNS;        // [kNS]
    uint64_t* s_full = v_empty + kNS;        // [kSB]
    uint64_t* p_full = s_full + kSB;         // [kSB]
    uint64_t* dq_done = p_full + kSB;
    uint64_t* dq_free = dq_done + 1;
    uint64_t* list_full = dq_free + 1;       // [2]
    uint64_t* list_empty = list_full + 2;    // [2]
    int* meta = reinterpret_cast<int*>(smem + L::kOffMeta);  // [2][4]: n, u, qb0, has2
    uint32_t* misc = reinterpret_cast<uint32_t*>(smem + L::kOffMisc);
    int32_t* lists = reinterpret_cast<int32_t*>(smem + L::kOffList);
    uint32_t* bm = reinterpret_cast<uint32_t*>(lists + 2 * p.max_list);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int n_frag = blockIdx.x < p.n_tiles ? (p.n_tiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;

    if (warp == 0 && lane == 0) {
        for (int i = 0; i < 2 + 4 * kNS + 2 * kSB + 6; ++i) mbar_init(bars + i, 1);
        for (int s = 0; s < kSB; ++s) mbar_init(p_full + s, kEw);
        mbar_init(q_full, kEw);  // Q / dO rows in TMEM, stored by the elementwise warps
        for (int s = 0; s < 2; ++s) mbar_init(list_empty + s, kEw + 1);
        mbar_init(dq_free, kEw);
        fence_barrier_init();
        tma_prefetch(&tm_q);
        tma_prefetch(&tm_do);
        tma_prefetch(&tm_k);
        tma_prefetch(&tm_v);
    }
    if (warp == 1) tmem_alloc<kBwdTmemCols>(misc);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = misc[0];
    pdl_wait();

    if (warp == 0) {
        // ================================================= list builder + TMA producer
        int jg = 0;
        for (int f = 0; f < n_frag; ++f) {
            const int lb = f & 1;
            mbar_wait(list_empty + lb, ((f >> 1) & 1) ^ 1);
            int32_t* list = lists + lb * p.max_list;
            const int tile = blockIdx.x + f * gridDim.x;
            const int u = tile / p.tiles_per_unit, qb0 = 2 * (tile % p.tiles_per_unit);
            const bool has2 = qb0 + 1 < p.nqb;
            for (int w = lane; w < 2 * p.bm_words; w += 32) bm[w] = 0u;
            __syncwarp();
            if (p.k > 0 && p.n_local > 0)
                for (int e = lane; e < (has2 ? 2 : 1) * p.k; e += 32) {
                    const int rw = e / p.k, c = e % p.k;
                    const int idx = __ldg(p.sel + (static_cast<int64_t>(u) * p.nqb + qb0 + rw) * p.k + c);
                    atomicOr(&bm[rw * p.bm_words + (idx >> 5)], 1u << (idx & 31));
                }
            for (int e = lane; e < p.n_dense; e += 32)
                list[e] = __ldg(p.dense + static_cast<int64_t>(u) * p.dense_stride + e) | (3 << 24);
            __syncwarp();
            int run = p.n_dense;
            const int32_t* loc = p.local + static_cast<int64_t>(u) * p.local_stride;
            for (int w0 = 0; w0 < p.bm_words; w0 += 32) {
                const int w = w0 + lane;
                const uint32_t a = w < p.bm_words ? bm[w] : 0u, c = w < p.bm_words ? bm[p.bm_words + w] : 0u;
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
                    list[pos++] = __ldg(loc + w * 32 + bit) |
                                  ((static_cast<int>((a >> bit) & 1u) | (static_cast<int>((c >> bit) & 1u) << 1)) << 24);
                }
                run += __shfl_sync(0xffffffffu, incl, 31);
            }
            if (lane == 0) {
                meta[lb * 4 + 0] = run;
                meta[lb * 4 + 1] = u;
                meta[lb * 4 + 2] = qb0;
                meta[lb * 4 + 3] = has2;
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(list_full + lb);
            const int nf = run;
            for (int idx = 0; idx < nf; ++idx) {
                const int j = jg + idx, s = j % kNS, ph = (j / kNS) & 1;
                const int row0 = (u * p.n_slots + (list[idx] & 0xFFFFFF)) * 64;
                mbar_wait(k_empty + s, ph ^ 1);
                if (elect_one()) {
                    mbar_arrive_expect_tx(k_full + s, L::kBlk);
                    for (int h = 0; h < L::kHalves; ++h) tma_load_2d(k_s + s * L::kBlk + h * 8192, &tm_k, k_full + s, h * 64, row0);
                }
                __syncwarp();
                mbar_wait(v_empty + s, ph ^ 1);
                if (elect_one()) {
                    mbar_arrive_expect_tx(v_full + s, L::kBlk);
                    for (int h = 0; h < L::kHalves; ++h) tma_load_2d(v_s + s * L::kBlk + h * 8192, &tm_v, v_full + s, h * 64, row0);
                }
                __syncwarp();
            }
            jg += nf;
        }
    } else if (warp == 1) {
        // ================================================= tcgen05 issuer
        constexpr uint32_t idesc_s = idesc_bf16_f32(128, 64, 0, 0);
        constexpr uint32_t idesc_o = idesc_bf16_f32(128, D, 0, 1);
        const uint64_t kdesc = smem_desc_sw128(smem_u32(k_s), 16, 1024);
        const uint64_t vdesc = smem_desc_sw128(smem_u32(v_s), 16, 1024);
        const uint64_t kmn = smem_desc_sw128(smem_u32(k_s), 8192, 1024);  // K as an MN-major B operand
        int jg = 0;
        for (int f = 0; f < n_frag; ++f) {
            const int lb = f & 1;
            mbar_wait(list_full + lb, (f >> 1) & 1);
            const int nf = meta[lb * 4];
            __syncwarp();
            if (lane == 0) mbar_arrive(list_empty + lb);
            if (f > 0) mbar_wait(dq_free, (f - 1) & 1);  // previous epilogue has read dQ
            mbar_wait(q_full, f & 1);
            tc_fence_after();
            auto issue_dq = [&](int x, bool first) {
                const int b = x % kSB;
                mbar_wait(p_full + b, (x / kSB) & 1);
                tc_fence_after();
                const uint32_t a_tmem = tmem + kBufCol + b * 128;  // dS_x (bf16 pairs) over S_x
                const uint64_t kd = kmn + (((x % kNS) * L::kBlk) >> 4);
                if (elect_one()) {
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk)
                        mma_ts(tmem, a_tmem + kA(kk), kd + ((kk * 2048) >> 4), idesc_o, (!first || kk > 0) ? 1u : 0u);
                    mma_commit(k_empty + x % kNS);
                }
                __syncwarp();
            };
            for (int idx = 0; idx < nf; ++idx) {
                const int j = jg + idx, s = j % kNS, b = j % kSB;
                mbar_wait(k_full + s, (j / kNS) & 1);
                mbar_wait(v_full + s, (j / kNS) & 1);
                tc_fence_after();
                const uint32_t st = tmem + kBufCol + b * 128, dpt = st + 64;
                const uint64_t kd = kdesc + ((s * L::kBlk) >> 4), vd = vdesc + ((s * L::kBlk) >> 4);
                if (elect_one()) {
#pragma unroll
                    for (int kk = 0; kk < D / 16; ++kk) {
                        const uint32_t oa = ((kk >> 2) * 16384 + (kk & 3) * 32) >> 4;
                        const uint32_t ob = ((kk >> 2) * 8192 + (kk & 3) * 32) >> 4;
                        (void)oa;
                        mma_ts(st, tmem + kQCol + kk * 8, kd + ob, idesc_s, kk > 0 ? 1u : 0u);
                        mma_ts(dpt, tmem + kDOCol + kk * 8, vd + ob, idesc_s, kk > 0 ? 1u : 0u);
                    }
                    mma_commit(v_empty + s);
                    mma_commit(s_full + b);
                }
                __syncwarp();
                if (idx >= kSB - 1) issue_dq(j - (kSB - 1), idx == kSB - 1);  // kSB - 1 blocks of lookahead
            }
            for (int x = (nf > kSB - 1 ? nf - (kSB - 1) : 0); x < nf; ++x) issue_dq(jg + x, x == 0);
            if (elect_one()) mma_commit(dq_done);
            __syncwarp();
            jg += nf;
        }
    } else {
        // ================================================= dS (thread = query row = TMEM lane)
        const int quarter = warp & 3, ch = (warp - 2) >> 2, r = quarter * 32 + lane, half = r >> 6, rr = r & 63;
        const uint32_t t_row = tmem + (static_cast<uint32_t>(quarter * 32) << 16);
        const float2 scl2 = make_float2(p.scale_log2, p.scale_log2);
        constexpr int DH = D / 2;  // dQ columns of this warp
        int jg = 0;
        for (int f = 0; f < n_frag; ++f) {
            const int lb = f & 1;
            mbar_wait(list_full + lb, (f >> 1) & 1);
            const int nf = meta[lb * 4], u = meta[lb * 4 + 1], qb0 = meta[lb * 4 + 2];
            const int32_t* list = lists + lb * p.max_list;
            const int qb = qb0 + half;
            const bool valid = rr < p.b && qb < p.nqb;
            const int64_t row = (static_cast<int64_t>(u) * p.nqb + qb) * p.b + rr;
            const int64_t prow = (static_cast<int64_t>(u) * p.nqb + qb) * 64 + rr;
            const float lse2 = valid ? __ldg(p.lse2 + prow) : INFINITY;
            const float dd = valid ? __ldg(p.drow + prow) : 0.0f;
            const float2 nl2 = make_float2(-lse2, -lse2);
            {   // this row's Q and dO (d columns [ch * D/2, +D/2)) into TMEM as bf16 pairs: the A
                // operands of the tile's S and dP MMAs (the previous tile's MMAs are complete:
                // its epilogue waited dq_done); padding rows are zero
                constexpr int W = D / 4;  // u32 per half row
                uint32_t qv[W], gv[W];
#pragma unroll
                for (int c = 0; c < W / 4; ++c) {
                    const uint4 a = valid ? __ldg(reinterpret_cast<const uint4*>(p.q + row * D + ch * (D / 2)) + c) : make_uint4(0, 0, 0, 0);
                    const uint4 g = valid ? __ldg(reinterpret_cast<const uint4*>(p.d_o + row * D + ch * (D / 2)) + c) : make_uint4(0, 0, 0, 0);
                    qv[4 * c] = a.x; qv[4 * c + 1] = a.y; qv[4 * c + 2] = a.z; qv[4 * c + 3] = a.w;
                    gv[4 * c] = g.x; gv[4 * c + 1] = g.y; gv[4 * c + 2] = g.z; gv[4 * c + 3] = g.w;
                }
                if constexpr (W == 32) {
                    tmem_st32(t_row + kQCol + ch * W, qv);
                    tmem_st32(t_row + kDOCol + ch * W, gv);
                } else {
                    tmem_st16(t_row + kQCol + ch * W, *reinterpret_cast<uint32_t(*)[16]>(qv));
                    tmem_st16(t_row + kDOCol + ch * W, *reinterpret_cast<uint32_t(*)[16]>(gv));
                }
                tmem_wait_st();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(q_full);
            }
            for (int idx = 0; idx < nf; ++idx) {
                const int j = jg + idx, b = j % kSB;
                mbar_wait(s_full + b, (j / kSB) & 1);
                tc_fence_after();
                const uint32_t ts = t_row + kBufCol + b * 128 + ch * 32;  // this warp's 32 key columns
                const bool vis = (list[idx] >> (24 + half)) & 1;
                uint32_t pk[16];
                if (vis) {
                    float sv[32], dp[32];
                    tmem_ld32(ts, *reinterpret_cast<uint32_t(*)[32]>(sv));
                    tmem_ld32(ts + 64, *reinterpret_cast<uint32_t(*)[32]>(dp));
                    tmem_wait_ld();
#pragma unroll
                    for (int c2 = 0; c2 < 16; ++c2) {
                        const int c = ch * 32 + 2 * c2;
                        const float2 x = __ffma2_rn(make_float2(sv[2 * c2], sv[2 * c2 + 1]), scl2, nl2);
                        const float p0 = c < p.b ? exp2_approx(x.x) : 0.0f;
                        const float p1 = c + 1 < p.b ? exp2_approx(x.y) : 0.0f;
                        pk[c2] = pack_bf16x2(p0 * (dp[2 * c2] - dd), p1 * (dp[2 * c2 + 1] - dd));
                    }
                } else {
#pragma unroll
                    for (int c = 0; c < 16; ++c) pk[c] = 0u;
                }
                tmem_st16(ts, pk);  // dS (bf16 pairs) over the fp32 S columns this warp read
                tmem_wait_st();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(p_full + b);
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(list_empty + lb);
            mbar_wait(dq_done, f & 1);
            tc_fence_after();
#pragma unroll 1
            for (int c0 = ch * DH; c0 < ch * DH + DH; c0 += 32) {
                uint32_t ov[32];
                if (nf > 0) {
                    tmem_ld32(t_row + c0, ov);
                    tmem_wait_ld();
                } else {
#pragma unroll
                    for (int c = 0; c < 32; ++c) ov[c] = 0u;
                }
                if (valid) {
#pragma unroll
                    for (int c = 0; c < 4; ++c) st_global_v8_scaled(p.dq + row * D + c0 + 8 * c, ov + 8 * c, p.scale);
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(dq_free);
            jg += nf;
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc<kBwdTmemCols>(tmem);
    }
}

// ---------------------------------------------------------------------------------- dK, dV
// Work item = (unit, pair of key blocks): dense pairs (dense[2i], dense[2i+1]) then local pairs
// (local[2i], local[2i+1]).  Rows 0-63 of the 128-row tile are slot A, 64-127 slot B.  The item's
// list = the query blocks that see A or B, with bit 0 / bit 1 = sees A / sees B.
template <int D>
__global__ void __launch_bounds__(kBwdThreads, 1)
    bwd_dkdv_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_do,
                    const __grid_constant__ CUtensorMap tm_k, const __grid_constant__ CUtensorMap tm_v,
                    const BwdParams p) {
    using L = BwdLayout<D>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* kp_s = smem + L::kOffA0;
    uint8_t* vp_s = smem + L::kOffA1;
    uint8_t* q_s = smem + L::kOffB;                   // [kNS] stages
    uint8_t* do_s = smem + L::kOffB + kNS * L::kBlk;  // [kNS] stages
    float* rows_s = reinterpret_cast<float*>(smem + L::kOffRow);  // [stage][lse2 | D][64]
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::kOffBar);
    uint64_t* kv_full = bars + 0;
    uint64_t* kv_empty = bars + 1;
    uint64_t* q_full = bars + 2;            // [kNS]
    uint64_t* q_empty = q_full + kNS;       // [kNS]
    uint64_t* s_full = q_empty + kNS;       // [2]
    uint64_t* p_full = s_full + 2;          // [2]
    uint64_t* acc_done = p_full + 2;
    uint64_t* acc_free = acc_done + 1;
    uint64_t* list_full = acc_free + 1;     // [2]
    uint64_t* list_empty = list_full + 2;   // [2]
    int* meta = reinterpret_cast<int*>(smem + L::kOffMeta);  // [2][4]: n, u, slot A, slot B (-1)
    uint32_t* misc = reinterpret_cast<uint32_t*>(smem + L::kOffMisc);
    int32_t* lists = reinterpret_cast<int32_t*>(smem + L::kOffList);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int n_frag = blockIdx.x < p.n_items ? (p.n_items - 1 - blockIdx.x) / gridDim.x + 1 : 0;

    if (warp == 0 && lane == 0) {
        for (int i = 0; i < 2 + 2 * kNS + 10; ++i) mbar_init(bars + i, 1);
        // a Q / dO / row stage is free once its MMAs completed (commit) AND the elementwise warps
        // have read its lse2 / D rows
        for (int s = 0; s < kNS; ++s) mbar_init(q_empty + s, 1 + kEw);
        for (int s = 0; s < 2; ++s) {
            mbar_init(p_full + s, kEw);
            mbar_init(list_empty + s, kEw + 1);
        }
        mbar_init(acc_free, kEw);
        fence_barrier_init();
        tma_prefetch(&tm_q);
        tma_prefetch(&tm_do);
        tma_prefetch(&tm_k);
        tma_prefetch(&tm_v);
    }
    if (warp == 1) tmem_alloc<kBwdTmemCols>(misc);
    if (warp >= 2) {  // Q / dO stages: rows >= b stay zero (finite operands for the masked columns)
        const int t = threadIdx.x - 64;
        for (int e = t; e < 2 * kNS * 64 * L::kHalves * 8; e += kEw * 32) {
            const int chunk = e & 7, rh = e >> 3;  // rh over [2 kNS stages][half][row 64]
            const int row = rh % 64, hs = rh / 64;
            if (row >= p.b) *reinterpret_cast<uint4*>(q_s + hs * 8192 + row * 128 + chunk * 16) = make_uint4(0, 0, 0, 0);
        }
        fence_proxy_async_smem();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = misc[0];
    pdl_wait();

    auto item_slots = [&](int item, int* u, int* sa, int* sb, int* la) {  // la: local index of A or -1
        const int per = p.dense_pairs + p.local_pairs;
        *u = item / per;
        const int pi = item % per;
        if (pi < p.dense_pairs) {
            const int32_t* dn = p.dense + static_cast<int64_t>(*u) * p.dense_stride;
            *sa = __ldg(dn + 2 * pi);
            *sb = 2 * pi + 1 < p.n_dense ? __ldg(dn + 2 * pi + 1) : -1;
            *la = -1;
        } else {
            const int li = 2 * (pi - p.dense_pairs);
            const int32_t* lc = p.local + static_cast<int64_t>(*u) * p.local_stride;
            *sa = __ldg(lc + li);
            *sb = li + 1 < p.n_local ? __ldg(lc + li + 1) : -1;
            *la = li;
        }
    };

    if (warp == 0) {
        // ================================================= list builder + TMA producer
        int jg = 0;
        for (int f = 0; f < n_frag; ++f) {
            const int lb = f & 1;
            mbar_wait(list_empty + lb, ((f >> 1) & 1) ^ 1);
            int32_t* list = lists + lb * p.max_list;
            int u, sa, sb, la;
            item_slots(blockIdx.x + f * gridDim.x, &u, &sa, &sb, &la);
            int run = 0;
            for (int i0 = 0; i0 < p.nqb; i0 += 32) {
                const int i = i0 + lane;
                int mask = 0;
                if (i < p.nqb) {
                    if (la < 0) {
                        mask = 1 | (sb >= 0 ? 2 : 0);
                    } else {
                        const uint32_t* ia = p.inv + (static_cast<int64_t>(u) * p.n_local + la) * p.inv_words;
                        mask = static_cast<int>((__ldg(ia + (i >> 5)) >> (i & 31)) & 1u);
                        if (sb >= 0) mask |= static_cast<int>((__ldg(ia + p.inv_words + (i >> 5)) >> (i & 31)) & 1u) << 1;
                    }
                }
                const uint32_t bal = __ballot_sync(0xffffffffu, mask != 0);
                if (mask) list[run + __popc(bal & ((1u << lane) - 1u))] = i | (mask << 24);
                run += __popc(bal);
            }
            if (lane == 0) {
                meta[lb * 4 + 0] = run;
                meta[lb * 4 + 1] = u;
                meta[lb * 4 + 2] = sa;
                meta[lb * 4 + 3] = sb;
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(list_full + lb);
            // the key/value pair (rows 0-63 slot A, 64-127 slot B; B absent -> stale rows, masked)
            if (f > 0) mbar_wait(kv_empty, (f - 1) & 1);
            if (elect_one()) {
                const uint32_t bytes = (sb >= 0 ? 2u : 1u) * L::kBlk;
                mbar_arrive_expect_tx(kv_full, 2 * bytes);
                for (int r = 0; r < (sb >= 0 ? 2 : 1); ++r) {
                    const int row0 = (u * p.n_slots + (r ? sb : sa)) * 64;
                    for (int h = 0; h < L::kHalves; ++h) {
                        tma_load_2d(kp_s + h * 16384 + r * 8192, &tm_k, kv_full, h * 64, row0);
                        tma_load_2d(vp_s + h * 16384 + r * 8192, &tm_v, kv_full, h * 64, row0);
                    }
                }
            }
            __syncwarp();
            const uint32_t qbytes = L::kHalves * static_cast<uint32_t>(p.b) * 128u;
            for (int idx = 0; idx < run; ++idx) {
                const int j = jg + idx, s = j % kNS;
                const int qb = list[idx] & 0xFFFFFF;
                mbar_wait(q_empty + s, ((j / kNS) & 1) ^ 1);
                if (elect_one()) {
                    mbar_arrive_expect_tx(q_full + s, 2 * qbytes + 2 * 256);
                    for (int h = 0; h < L::kHalves; ++h) {
                        tma_load_3d(q_s + s * L::kBlk + h * 8192, &tm_q, q_full + s, h * 64, 0, u * p.nqb + qb);
                        tma_load_3d(do_s + s * L::kBlk + h * 8192, &tm_do, q_full + s, h * 64, 0, u * p.nqb + qb);
                    }
                    const int64_t r0 = (static_cast<int64_t>(u) * p.nqb + qb) * 64;
                    bulk_g2s(rows_s + s * 128, p.lse2 + r0, 256, q_full + s);
                    bulk_g2s(rows_s + s * 128 + 64, p.drow + r0, 256, q_full + s);
                }
                __syncwarp();
            }
            jg += run;
        }
    } else if (warp == 1) {
        // ================================================= tcgen05 issuer
        constexpr uint32_t idesc_s = idesc_bf16_f32(128, 64, 0, 0);
        constexpr uint32_t idesc_o = idesc_bf16_f32(128, D, 0, 1);
        const uint64_t kdesc = smem_desc_sw128(smem_u32(kp_s), 16, 1024);
        const uint64_t vdesc = smem_desc_sw128(smem_u32(vp_s), 16, 1024);
        const uint64_t qdesc = smem_desc_sw128(smem_u32(q_s), 16, 1024);
        const uint64_t dodesc = smem_desc_sw128(smem_u32(do_s), 16, 1024);
        const uint64_t qmn = smem_desc_sw128(smem_u32(q_s), 8192, 1024);
        const uint64_t domn = smem_desc_sw128(smem_u32(do_s), 8192, 1024);
        int jg = 0;
        for (int f = 0; f < n_frag; ++f) {
            const int lb = f & 1;
            mbar_wait(list_full + lb, (f >> 1) & 1);
            const int nf = meta[lb * 4];
            __syncwarp();
            if (lane == 0) mbar_arrive(list_empty + lb);
            if (f > 0) mbar_wait(acc_free, (f - 1) & 1);  // previous epilogue has read dK / dV
            mbar_wait(kv_full, f & 1);
            tc_fence_after();
            auto issue_acc = [&](int x, bool first) {
                const int b = x & 1, sx = x % kNS;
                mbar_wait(p_full + b, (x >> 1) & 1);
                bstamp(p, 2, x);  // MMA: P_x seen
                tc_fence_after();
                const uint32_t pt = tmem + 256 + b * 128, dst = pt + 64;  // P^T, dS^T (bf16 pairs)
                const uint64_t qd = qmn + ((sx * L::kBlk) >> 4), dd = domn + ((sx * L::kBlk) >> 4);
                if (elect_one()) {
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk) {
                        mma_ts(tmem + 128, pt + kA(kk), dd + ((kk * 2048) >> 4), idesc_o, (!first || kk > 0) ? 1u : 0u);
                        mma_ts(tmem, dst + kA(kk), qd + ((kk * 2048) >> 4), idesc_o, (!first || kk > 0) ? 1u : 0u);
                    }
                    mma_commit(q_empty + sx);
                }
                __syncwarp();
                bstamp(p, 3, x);  // MMA: dV / dK of x issued
            };
            for (int idx = 0; idx < nf; ++idx) {
                const int j = jg + idx, s = j % kNS, b = j & 1;
                mbar_wait(q_full + s, (j / kNS) & 1);
                bstamp(p, 0, j);  // MMA: Q_j / dO_j present, before S_j
                tc_fence_after();
                const uint32_t st = tmem + 256 + b * 128, dpt = st + 64;
                const uint64_t qd = qdesc + ((s * L::kBlk) >> 4), dd = dodesc + ((s * L::kBlk) >> 4);
                if (elect_one()) {
#pragma unroll
                    for (int kk = 0; kk < D / 16; ++kk) {
                        const uint32_t oa = ((kk >> 2) * 16384 + (kk & 3) * 32) >> 4;
                        const uint32_t ob = ((kk >> 2) * 8192 + (kk & 3) * 32) >> 4;
                        mma_ss(st, kdesc + oa, qd + ob, idesc_s, kk > 0 ? 1u : 0u);
                        mma_ss(dpt, vdesc + oa, dd + ob, idesc_s, kk > 0 ? 1u : 0u);
                    }
                    mma_commit(s_full + b);
                }
                __syncwarp();
                bstamp(p, 1, j);  // MMA: S_j, dP_j issued
                if (idx > 0) issue_acc(j - 1, idx == 1);
            }
            if (nf > 0) issue_acc(jg + nf - 1, nf == 1);
            if (elect_one()) {
                mma_commit(kv_empty);
                mma_commit(acc_done);
            }
            __syncwarp();
            jg += nf;
        }
    } else {
        // ================================================= P^T, dS^T (thread = key row = TMEM lane)
        const int quarter = warp & 3, ch = (warp - 2) >> 2, r = quarter * 32 + lane, half = r >> 6, rr = r & 63;
        const uint32_t t_row = tmem + (static_cast<uint32_t>(quarter * 32) << 16);
        constexpr int DH = D / 2;
        int jg = 0;
        for (int f = 0; f < n_frag; ++f) {
            const int lb = f & 1;
            mbar_wait(list_full + lb, (f >> 1) & 1);
            const int nf = meta[lb * 4], u = meta[lb * 4 + 1], sa = meta[lb * 4 + 2], sb = meta[lb * 4 + 3];
            const int32_t* list = lists + lb * p.max_list;
            const int slot = half ? sb : sa;
            const bool kvalid = rr < p.b && slot >= 0;
            for (int idx = 0; idx < nf; ++idx) {
                const int j = jg + idx, bb = j & 1, s = j % kNS;
                if (threadIdx.x == 64) bstamp(p, 4, j);  // elementwise warp 2: waiting for S_j
                mbar_wait(s_full + bb, (j >> 1) & 1);
                if (threadIdx.x == 64) bstamp(p, 5, j);  // S_j seen
                tc_fence_after();
                const uint32_t ts = t_row + 256 + bb * 128 + ch * 32;  // this warp's 32 query columns
                const bool vis = (list[idx] >> (24 + half)) & 1;
                uint32_t pp[16], pd[16];
                if (vis) {
                    float sv[32], dp[32];
                    tmem_ld32(ts, *reinterpret_cast<uint32_t(*)[32]>(sv));
                    tmem_ld32(ts + 64, *reinterpret_cast<uint32_t(*)[32]>(dp));
                    // the lse2 / D rows of stage s arrived with q_full[s] (bulk copy): acquire that
                    // phase here too (already complete -- S_j was issued after it -- so this is
                    // ordering, not waiting; the stage is reloaded only after q_empty[s], which
                    // counts this warp's arrival below)
                    mbar_wait(q_full + s, (j / kNS) & 1);
                    tmem_wait_ld();
                    const float* l2 = rows_s + s * 128 + ch * 32;
                    const float* dd = l2 + 64;
#pragma unroll
                    for (int c2 = 0; c2 < 16; ++c2) {
                        const int c = ch * 32 + 2 * c2;
                        const float2 lq = *reinterpret_cast<const float2*>(l2 + 2 * c2);
                        const float2 dq = *reinterpret_cast<const float2*>(dd + 2 * c2);
                        const float x0 = fmaf(sv[2 * c2], p.scale_log2, -lq.x), x1 = fmaf(sv[2 * c2 + 1], p.scale_log2, -lq.y);
                        const float p0 = (kvalid && c < p.b) ? exp2_approx(x0) : 0.0f;
                        const float p1 = (kvalid && c + 1 < p.b) ? exp2_approx(x1) : 0.0f;
                        pp[c2] = pack_bf16x2(p0, p1);
                        pd[c2] = pack_bf16x2(p0 * (dp[2 * c2] - dq.x), p1 * (dp[2 * c2 + 1] - dq.y));
                    }
                } else {
#pragma unroll
                    for (int c = 0; c < 16; ++c) pp[c] = pd[c] = 0u;
                }
                tmem_st16(ts, pp);
                tmem_st16(ts + 64, pd);
                tmem_wait_st();
                tc_fence_before();
                __syncwarp();
                if (threadIdx.x == 64) bstamp(p, 6, j);  // P_j arrive
                if (lane == 0) {
                    mbar_arrive(p_full + bb);
                    mbar_arrive(q_empty + s);  // this warp is done with the stage's rows
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(list_empty + lb);
            if (threadIdx.x == 64) bstamp(p, 7, f);  // fragment f: waiting for the accumulators
            mbar_wait(acc_done, f & 1);
            if (threadIdx.x == 64) bstamp(p, 8, f);  // accumulators complete, epilogue starts
            tc_fence_after();
            // dK = scale * acc[0, D), dV = acc[128, 128 + D): this warp's column half of its rows
#pragma unroll 1
            for (int which = 0; which < 2; ++which) {
                float* outp = which ? p.dv : p.dk;
                const float mul = which ? 1.0f : p.scale;
#pragma unroll 1
                for (int c0 = ch * DH; c0 < ch * DH + DH; c0 += 32) {
                    uint32_t ov[32];
                    if (nf > 0) {
                        tmem_ld32(t_row + which * 128 + c0, ov);
                        tmem_wait_ld();
                    } else {
#pragma unroll
                        for (int c = 0; c < 32; ++c) ov[c] = 0u;
                    }
                    if (kvalid) {
                        float* dst = outp + ((static_cast<int64_t>(u) * p.n_slots + slot) * 64 + rr) * D + c0;
#pragma unroll
                        for (int c = 0; c < 4; ++c) st_global_v8_scaled(dst + 8 * c, ov + 8 * c, mul);
                    }
                }
            }
            tc_fence_before();
            __syncwarp();
            if (threadIdx.x == 64) bstamp(p, 9, f);  // epilogue done
            if (lane == 0) mbar_arrive(acc_free);
            jg += nf;
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc<kBwdTmemCols>(tmem);
    }
}

template <int D>
int launch_bwd_impl(const bf16* q, const bf16* kp, const bf16* vp, const bf16* d_o, BwdParams p, cudaStream_t s) {
    using L = BwdLayout<D>;
    alignas(64) CUtensorMap tq, tdo, tk, tv;
    std::string err;
    {
        const uint64_t dims[3] = {static_cast<uint64_t>(D), static_cast<uint64_t>(p.b),
                                  static_cast<uint64_t>(p.units) * p.nqb};
        const uint64_t strides[2] = {static_cast<uint64_t>(D) * 2, static_cast<uint64_t>(p.b) * D * 2};
        const uint32_t box[3] = {64, static_cast<uint32_t>(p.b), 1};
        if (!encode_tmap_bf16(&tq, q, 3, dims, strides, box, &err) || !encode_tmap_bf16(&tdo, d_o, 3, dims, strides, box, &err))
            return set_error(PBSA_ECUDA, "bsa_bwd: tensor map Q/dO: " + err);
    }
    {
        const uint64_t dims[2] = {static_cast<uint64_t>(D), static_cast<uint64_t>(p.units) * p.n_slots * 64};
        const uint64_t strides[1] = {static_cast<uint64_t>(D) * 2};
        const uint32_t box[2] = {64, 64};
        if (!encode_tmap_bf16(&tk, kp, 2, dims, strides, box, &err) || !encode_tmap_bf16(&tv, vp, 2, dims, strides, box, &err))
            return set_error(PBSA_ECUDA, "bsa_bwd: tensor map K/V: " + err);
    }
    const size_t smem = L::bytes(p.max_list, p.bm_words);
    if (smem > 227 * 1024) return set_error(PBSA_EUNSUPPORTED, "bsa_bwd: visible list too long for shared memory");
    int sms = 0, dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (p.n_tiles > 0) {
        if (int rc = ensure_smem(reinterpret_cast<const void*>(bwd_dq_kernel<D>), smem, "bsa_bwd dq")) return rc;
        const int grid = p.n_tiles < sms ? p.n_tiles : sms;
        if (launch_pdl(bwd_dq_kernel<D>, dim3(grid), dim3(kBwdThreads), smem, s, tq, tdo, tk, tv, p) != cudaSuccess)
            return check_launch("bwd_dq_kernel");
    }
    if (p.n_items > 0) {
        if (int rc = ensure_smem(reinterpret_cast<const void*>(bwd_dkdv_kernel<D>), smem, "bsa_bwd dkdv")) return rc;
        const int grid = p.n_items < sms ? p.n_items : sms;
        if (launch_pdl(bwd_dkdv_kernel<D>, dim3(grid), dim3(kBwdThreads), smem, s, tq, tdo, tk, tv, p) != cudaSuccess)
            return check_launch("bwd_dkdv_kernel");
    }
    return check_launch("bsa_bwd");
}

}  // namespace

size_t bsa_bwd_workspace(int units, int nqb, int b, int n_local) {
    (void)b;
    const size_t rows = static_cast<size_t>(units) * nqb * 64;
    const size_t words = (static_cast<size_t>(nqb) + 31) / 32;
    return 2 * rows * 4 + static_cast<size_t>(units) * n_local * words * 4 + 256;
}

static long long* g_bwd_trace = nullptr;  // perf experiments: dK/dV handshake timeline (CTA 0)

int launch_bsa_bwd(const bf16* q, const bf16* k_pool, const bf16* v_pool, int n_slots, const int32_t* dense,
                   int dense_stride, int n_dense, const int32_t* local, int local_stride, int n_local,
                   const int32_t* sel, int k, int nqb, int b, int d, int units, float scale, const bf16* o,
                   const bf16* d_o, const float* lse, float* dq, float* dk, float* dv, void* ws, size_t ws_bytes,
                   cudaStream_t s) {
    if (units == 0 || nqb == 0) return 0;
    if (ws_bytes < bsa_bwd_workspace(units, nqb, b, n_local)) return set_error(PBSA_EINVAL, "bsa_bwd: workspace too small");
    BwdParams p{};
    p.trace = g_bwd_trace;
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
    p.k = n_local > 0 ? k : 0;
    p.scale = scale;
    p.scale_log2 = scale * 1.4426950408889634f;
    const int64_t rows = static_cast<int64_t>(units) * nqb * b;
    float* lse2 = static_cast<float*>(ws);
    float* drow = lse2 + static_cast<int64_t>(units) * nqb * 64;
    uint32_t* inv = reinterpret_cast<uint32_t*>(drow + static_cast<int64_t>(units) * nqb * 64);
    p.lse2 = lse2;
    p.drow = drow;
    p.inv = inv;
    p.inv_words = (nqb + 31) / 32;
    p.q = q;
    p.d_o = d_o;
    p.dq = dq;
    p.dk = dk;
    p.dv = dv;
    p.bm_words = (n_local + 31) / 32 + 1;
    p.max_list = n_dense + (p.k > 0 ? (2 * p.k < n_local ? 2 * p.k : n_local) : 0);
    if (p.max_list < nqb) p.max_list = nqb;  // the dK/dV lists hold query blocks
    p.tiles_per_unit = (nqb + 1) / 2;
    p.n_tiles = units * p.tiles_per_unit;
    p.dense_pairs = (n_dense + 1) / 2;
    p.local_pairs = p.k > 0 ? (n_local + 1) / 2 : 0;
    p.n_items = units * (p.dense_pairs + p.local_pairs);
    // D = rowsum(dO o O), lse * log2(e); zero padding rows read by the 64-row staging copies
    if (cudaMemsetAsync(ws, 0, ws_bytes, s) != cudaSuccess) return check_launch("bsa_bwd memset");
    launch_pdl(bwd_rows_kernel, dim3(static_cast<unsigned>((rows + 7) / 8)), dim3(256), 0, s, o, d_o, lse, rows, d, b,
               lse2, drow);
    if (p.local_pairs > 0) {
        const int64_t n = static_cast<int64_t>(units) * nqb * p.k;
        launch_pdl(bwd_inv_kernel, dim3(static_cast<unsigned>((n + 255) / 256)), dim3(256), 0, s, sel, units, nqb, p.k,
                   n_local, p.inv_words, inv);
    }
    if (int rc = check_launch("bsa_bwd prep")) return rc;
    if (d == 128) return launch_bwd_impl<128>(q, k_pool, v_pool, d_o, p, s);
    return launch_bwd_impl<64>(q, k_pool, v_pool, d_o, p, s);
}

}  // namespace pbsa

extern "C" void pbsa_debug_bwd_trace_buffer(void* p) { pbsa::g_bwd_trace = static_cast<long long*>(p); }
