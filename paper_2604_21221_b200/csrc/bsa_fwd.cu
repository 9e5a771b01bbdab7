// bsa_fwd.cu -- K3 block-sparse attention forward on tcgen05 / TMEM / TMA (sm_100a).
//
// Reference op: attention.attention_sparse: for each query block, softmax over
// the persistent blocks + current chunk (dense, Eq. 5) and the Top-K selected
// local blocks (Eq. 11), online softmax; masked blocks are never loaded.
//
// Tile: 128 query rows = two consecutive query blocks (rows [0,64) hold block 2t, [64,128) block
// 2t+1; rows >= b of each half are zero padding).  M=128 is the full-rate tcgen05 shape (M=64 per
// query block would issue at half rate).  The tile walks the UNION of both blocks' visible key
// blocks -- dense blocks first, then the union of the two Top-K selections (built from two
// bitmaps) -- with a 2-bit mask per entry saying which half sees it.
//
// Schedule (persistent, 2 CTAs per SM).  Without a workspace every CTA takes whole tiles
// round-robin (tile = cta + f * grid).  With one (hybrid stream-K): full waves of whole tiles
// first -- concurrently active tiles then belong to few heads, whose KV blocks stay L2-resident
// -- and only the tail tiles (n_tiles mod grid) are split: their iteration space (tile x virtual
// visible-block index, every tile counted with the upper-bound length V) is cut into equal
// contiguous ranges, one per tail CTA, so a CTA processes at most two tile FRAGMENTS of the
// tail.  A fragment writes fp32 partials (unnormalised O, running max m, sum l) to a workspace;
// once a CTA has finished all its fragments it waits for the other fragments of each split tile
// it holds (per-tile arrival counter) and merges ITS SLICE of the tile's rows, in fragment order
// (deterministic) -- the nf CTAs of a tile merge it in parallel (a single last-arriving merger was
// a 20-38 us serial tail per launch).  This removes the 1.58-wave quantisation of one-tile-per-CTA
// launches at the Wan-1.3B shape (468 tiles on 296 CTA slots).
//
// Warp roles (192 threads):
//   warp 0  TMA producer: Q (3-D map over [unit*nqb][b][d], one box per query block and d-half),
//           K and V slots (2-D maps over the slot pools, one 64x64 box per d-half)
//   warp 1  tcgen05 issuer: S_j = Q K_j^T (SS, M128 N64), O += P_j V_j (TS: P from TMEM as packed
//           bf16, V as an MN-major operand), commits to mbarriers
//   warps 2-5  softmax: thread = query row = TMEM lane; online softmax with lazy
//           rescale (only when the running max grows by > 8 in log2 units), P written back over
//           S in TMEM; epilogue O / l straight from TMEM to HBM (or to the partial workspace).
// TMEM: O [0, d), S0 [d, d+64), S1 [d+64, d+128) -> 256 columns, two CTAs per SM.
//
// Roofline: tensor core.  Executed FLOPs per tile = 4 * 128 * 64 * d * |union list|.
#include <cfloat>
#include <cstdio>
#include <cstdlib>

#include "bsa_common.cuh"
#include "internal.h"
#include "ptx.cuh"

namespace pbsa {
namespace {

constexpr int kThreads = 192;
template <int D, int NSK, int NSV>
struct Layout {
    static constexpr int kHalves = D / 64;
    static constexpr uint32_t kQBytes = kHalves * 128 * 128;  // [half][128 rows][128 B]
    static constexpr uint32_t kKVBytes = kHalves * 64 * 128;  // one slot: [half][64 rows][128 B]
    static constexpr uint32_t kOffQ = 0;
    static constexpr uint32_t kOffK = kOffQ + kQBytes;
    static constexpr uint32_t kOffV = kOffK + NSK * kKVBytes;
    static constexpr uint32_t kOffBar = kOffV + NSV * kKVBytes;
    // q_full, q_empty, k_full/empty[NSK], v_full/empty[NSV], s_full[2], p_full[2], o_done[2],
    // o_free, list_full[2], list_empty[2], merge
    static constexpr int kNumBars = 2 + 2 * NSK + 2 * NSV + 6 + 1 + 4 + 1;
    static constexpr uint32_t kOffMeta = kOffBar + kNumBars * 8;
    static constexpr uint32_t kOffMisc = kOffMeta + 2 * sizeof(FragMeta);
    static constexpr uint32_t kOffList = kOffMisc + 16;
    static constexpr uint32_t kSColBase = D;  // S0 at D, S1 at D + 64
    static size_t bytes(int max_list, int bm_words, int entry_bytes) {
        const size_t lb = (2 * static_cast<size_t>(max_list) * entry_bytes + 15) & ~size_t(15);
        return 1024 + kOffList + lb + 2 * static_cast<size_t>(bm_words) * 4;
    }
};

// handshake timeline (tools/k3_timeline.py): compiled in only with -DPBSA_K3_TRACE
__device__ __forceinline__ void stamp(const BsaParams& p, int ev, int j) {
#ifdef PBSA_K3_TRACE
    if (p.trace != nullptr && blockIdx.x == 0 && j < 256) p.trace[ev * 256 + j] = clock64();
#else
    (void)p; (void)ev; (void)j;
#endif
}
// per-CTA milestones on the global timer (tools/k3_cta_timeline.py), same build flag:
// trace[15 * 256 + cta * 8 + ev], ev 0 start / 1 first list built / 2 first S seen / 3 last P
// arrived / 4 partial written / 5 merge start / 6 merge end / 7 exit (slot 7 also gets the SM id)
__device__ __forceinline__ void stamp_cta(const BsaParams& p, int ev) {
#ifdef PBSA_K3_TRACE
    if (p.trace != nullptr) {
        uint64_t t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        p.trace[15 * 256 + blockIdx.x * 8 + ev] = static_cast<long long>(t);
    }
#else
    (void)p; (void)ev;
#endif
}

template <int D, int NSK, int NSV, int B, uint32_t POLY, bool L16>
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
    uint64_t* q_empty = bars + 1;
    uint64_t* k_full = bars + 2;
    uint64_t* k_empty = k_full + NSK;
    uint64_t* v_full = k_empty + NSK;
    uint64_t* v_empty = v_full + NSV;
    uint64_t* s_full = v_empty + NSV;
    uint64_t* p_full = s_full + 2;
    uint64_t* o_done = p_full + 2;
    uint64_t* o_free = o_done + 2;
    uint64_t* list_full = o_free + 1;
    uint64_t* list_empty = list_full + 2;
    uint64_t* merge_bar = list_empty + 2;
    FragMeta* meta = reinterpret_cast<FragMeta*>(smem + L::kOffMeta);
    uint32_t* misc = reinterpret_cast<uint32_t*>(smem + L::kOffMisc);  // [0] tmem base
    // visible lists, double-buffered: [2][max_list] entries of 4 bytes (slot | mask << 24) or, when
    // the pool has < 16384 slots, 2 bytes (slot | mask << 14) -- halves the footprint of long lists
    // (config 5: 3238 entries) so two CTAs still fit an SM
    uint8_t* lists = smem + L::kOffList;
    constexpr int esz = L16 ? 2 : 4;
    constexpr int mshift = L16 ? 14 : 24;
    uint32_t* bm = reinterpret_cast<uint32_t*>(lists + ((2 * static_cast<size_t>(p.max_list) * esz + 15) & ~size_t(15)));
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int cta = blockIdx.x;
    const int n_frag = num_fragments(p, cta);

    // ------------------------------------------------------------------ setup
    if (warp == 0 && lane == 0) {
        mbar_init(q_full, 1);
        mbar_init(q_empty, 1);
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
            mbar_init(p_full + s, 4);  // one elected arrival per softmax warp
            mbar_init(o_done + s, 1);
            mbar_init(list_full + s, 1);
            mbar_init(list_empty + s, 5);  // MMA warp + 4 softmax warps
        }
        mbar_init(o_free, 4);
        mbar_init(merge_bar, 1);
        fence_barrier_init();
        tma_prefetch(&tm_q);
        tma_prefetch(&tm_k);
        tma_prefetch(&tm_v);
    }
    if (warp == 1) tmem_alloc<kTmemCols>(misc);
    if (warp >= 2) {
        // zero all query padding rows once: TMA only ever writes rows < b of each half, so the
        // padding stays zero (finite S) for every tile this CTA processes
        const int t = threadIdx.x - 64;
        for (int e = t; e < 128 * L::kHalves * 8; e += 128) {
            const int chunk = e & 7, rh = e >> 3;
            const int h = rh % L::kHalves, row = rh / L::kHalves;
            if ((row & 63) >= p.b)
                *reinterpret_cast<uint4*>(q_smem + h * 16384 + row * 128 + chunk * 16) = make_uint4(0, 0, 0, 0);
        }
        // likewise the rows >= b of every K and V ring slot: the K/V boxes carry the b valid rows of a
        // pool slot only (6 % less L2 -> SM traffic at b = 60); zero rows keep S finite and P V exact
        for (int e = t; e < (NSK + NSV) * L::kHalves * 64 * 8; e += 128) {
            const int chunk = e & 7, row = (e >> 3) & 63, sh = e >> 9;  // sh = ring slot * kHalves + half
            if (row >= p.b)
                *reinterpret_cast<uint4*>(k_smem + sh * 8192 + row * 128 + chunk * 16) = make_uint4(0, 0, 0, 0);
        }
        fence_proxy_async_smem();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = misc[0];
    // programmatic dependent launch: everything above (barriers, TMEM, tensor-map prefetch, Q
    // padding) overlapped the previous kernel; its outputs (selections, Q) are visible from here
    pdl_wait();
    if (threadIdx.x == 0) stamp_cta(p, 0);

    if (warp == 0) {
        // ============================================================== TMA producer
        // whole warp in the loop (uniform operands), one elected lane issues each TMA
        {
            // The producer also builds each fragment's visible list (double-buffered): list f+1 is
            // built while the MMA / softmax warps still work on the last blocks of fragment f.
            int jg = 0, q_uses = 0;
            // a K / V box covers the slot's b valid rows only (rows >= b of the ring slots were zeroed
            // at setup and are never written by TMA)
            const uint32_t kv_tx = static_cast<uint32_t>(L::kHalves) * static_cast<uint32_t>(p.b) * 128u;
            for (int f = 0; f < n_frag; ++f) {
                const int lb = f & 1;
                mbar_wait(list_empty + lb, ((f >> 1) & 1) ^ 1);
                uint8_t* list = lists + static_cast<size_t>(lb) * p.max_list * esz;
                // ---------------------------------------------------------- fragment schedule
                const FragPlan fp = plan_fragment(p, cta, f);
                gang_wait(p, cta, f);  // unit gangs: every member has issued the previous unit's loads
                // ---------------------------------------------------------- visible list of the tile
                const int run = build_visible_list<L16>(p, fp, list, bm);
                const FragMeta fm = make_meta(p, fp, run);
                if (lane == 0) meta[lb] = fm;
                if (lane == 0 && f == 0) stamp_cta(p, 1);
                __syncwarp();
                if (lane == 0) mbar_arrive(list_full + lb);
                const int nf = fm.e1 - fm.e0;
                if (nf > 0) {
                    if (q_uses > 0) mbar_wait(q_empty, (q_uses - 1) & 1);
                    const uint32_t qbytes = (fm.qb1 >= 0 ? 2u : 1u) * L::kHalves * static_cast<uint32_t>(p.b) * 128u;
                    if (elect_one()) {
                        mbar_arrive_expect_tx(q_full, qbytes);
                        for (int r = 0; r < (fm.qb1 >= 0 ? 2 : 1); ++r)
                            for (int h = 0; h < L::kHalves; ++h) {
                                if (p.lat) {  // the query block is one 5-D box of the latent (blockify)
                                    const int qb = r ? fm.qb1 : fm.qb0, e = fm.u / p.lg.heads, hd = fm.u % p.lg.heads;
                                    const int nw = qb % p.lg.nw(), nh = (qb / p.lg.nw()) % p.lg.nh();
                                    const int nt = qb / (p.lg.nw() * p.lg.nh());
                                    tma_load_5d(q_smem + h * 16384 + r * 8192, &tm_q, q_full, hd * D + h * 64,
                                                nw * p.lg.bw, nh * p.lg.bh, nt * p.lg.bt, e);
                                } else {
                                    tma_load_3d(q_smem + h * 16384 + r * 8192, &tm_q, q_full, h * 64, 0,
                                                fm.u * p.nqb + (r ? fm.qb1 : fm.qb0));
                                }
                            }
                    }
                    __syncwarp();
                    ++q_uses;
                    auto load_v = [&](int idx) {
                        const int j = jg + idx;
                        const int s = j % NSV;
                        mbar_wait(v_empty + s, ((j / NSV) & 1) ^ 1);
                        const int row0 = (fm.u * p.n_slots + list_slot<L16>(list, fm.e0 + idx)) * 64;
                        if (elect_one()) {
                            if (p.ablate & 2) {  // experiment: no K/V traffic
                                mbar_arrive(v_full + s);
                            } else {
                                mbar_arrive_expect_tx(v_full + s, kv_tx);
                                for (int h = 0; h < L::kHalves; ++h)
                                    tma_load_2d(v_smem + s * L::kKVBytes + h * 8192, &tm_v, v_full + s, h * 64, row0);
                            }
                        }
                        __syncwarp();
                    };
                    for (int idx = 0; idx < nf; ++idx) {
                        const int j = jg + idx;
                        const int s = j % NSK;
                        mbar_wait(k_empty + s, ((j / NSK) & 1) ^ 1);
                        const int row0 = (fm.u * p.n_slots + list_slot<L16>(list, fm.e0 + idx)) * 64;
                        if (elect_one()) {
                            if (p.ablate & 2) {
                                mbar_arrive(k_full + s);
                            } else {
                                mbar_arrive_expect_tx(k_full + s, kv_tx);
                                for (int h = 0; h < L::kHalves; ++h)
                                    tma_load_2d(k_smem + s * L::kKVBytes + h * 8192, &tm_k, k_full + s, h * 64, row0);
                            }
                        }
                        __syncwarp();
                        if (idx >= 1) load_v(idx - 1);
                    }
                    load_v(nf - 1);
                    jg += nf;
                }
                gang_arrive(p, cta, f);
            }
        }
    } else if (warp == 1) {
        // ============================================================== tcgen05 issuer
        // The whole warp runs the loop so every descriptor is warp-uniform (uniform registers,
        // no per-instruction R2UR); one lane issues each tcgen05 instruction.
        {
            constexpr uint32_t idesc_s = idesc_bf16_f32(128, 64, 0, 0);
            constexpr uint32_t idesc_o = idesc_bf16_f32(128, D, 0, 1);
            const bool do_mma = (p.ablate & 4) == 0;
            const uint64_t qdesc = smem_desc_sw128(smem_u32(q_smem), 16, 1024);
            const uint64_t kdesc = smem_desc_sw128(smem_u32(k_smem), 16, 1024);
            const uint64_t vdesc = smem_desc_sw128(smem_u32(v_smem), 8192, 1024);
            int jg = 0, q_uses = 0;
            auto issue_s = [&](int j) {
                const int s = j % NSK;
                mbar_wait(k_full + s, (j / NSK) & 1);
                tc_fence_after();
                const uint32_t d_tmem = tmem + L::kSColBase + (j & 1) * 64;
                const uint64_t kd = kdesc + ((s * L::kKVBytes) >> 4);
                if (elect_one()) {
                    if (do_mma) {
#pragma unroll
                        for (int kk = 0; kk < D / 16; ++kk) {
                            const uint32_t off_q = ((kk >> 2) * 16384 + (kk & 3) * 32) >> 4;
                            const uint32_t off_k = ((kk >> 2) * 8192 + (kk & 3) * 32) >> 4;
                            mma_ss(d_tmem, qdesc + off_q, kd + off_k, idesc_s, kk > 0 ? 1u : 0u);
                        }
                    }
                    mma_commit(k_empty + s);
                    mma_commit(s_full + (j & 1));
                }
                __syncwarp();
            };
            for (int f = 0; f < n_frag; ++f) {
                const int lb = f & 1;
                mbar_wait(list_full + lb, (f >> 1) & 1);
                const int nf = meta[lb].e1 - meta[lb].e0;
                __syncwarp();
                if (lane == 0) mbar_arrive(list_empty + lb);
                if (f > 0) mbar_wait(o_free, (f - 1) & 1);  // previous epilogue has read O
                if (nf == 0) continue;
                mbar_wait(q_full, q_uses & 1);
                tc_fence_after();
                issue_s(jg);
                for (int idx = 0; idx < nf; ++idx) {
                    const int j = jg + idx;
                    stamp(p, 0, j);  // MMA: before issuing S_{j+1}
                    if (idx + 1 < nf) issue_s(j + 1);
                    const int sv = j % NSV;
                    stamp(p, 1, j);  // MMA: S_{j+1} issued, waiting for P_j
                    mbar_wait(p_full + (j & 1), (j >> 1) & 1);
                    stamp(p, 2, j);  // MMA: P_j seen
                    mbar_wait(v_full + sv, (j / NSV) & 1);
                    tc_fence_after();
                    const uint32_t a_tmem = tmem + L::kSColBase + (j & 1) * 64;
                    const uint64_t vd = vdesc + ((sv * L::kKVBytes) >> 4);
                    if (elect_one()) {
                        if (do_mma) {
#pragma unroll
                            for (int kk = 0; kk < 4; ++kk)
                                mma_ts(tmem, a_tmem + kk * 8, vd + ((kk * 2048) >> 4), idesc_o,
                                       (idx > 0 || kk > 0) ? 1u : 0u);
                        }
                        mma_commit(v_empty + sv);
                        mma_commit(o_done + (j & 1));
                    }
                    __syncwarp();
                    stamp(p, 3, j);  // MMA: PV_j issued
                }
                if (elect_one()) mma_commit(q_empty);  // every S MMA reading this Q has been issued
                __syncwarp();
                ++q_uses;
                jg += nf;
            }
        }
    } else {
        // ============================================================== softmax
        const int t = threadIdx.x - 64;
        const int quarter = warp & 3;
        const int r = quarter * 32 + lane;
        const int half = r >> 6, rr = r & 63;
        const uint32_t lane_base = static_cast<uint32_t>(quarter * 32) << 16;
        const uint32_t t_o = tmem + lane_base;
        // Wait until PV_x has completed.  o_done[x & 1] completes once per PV of that parity; PV_x
        // is the LATEST PV of its parity that can have been issued when this is called (PV_{x+2}
        // needs P_{x+2}, which this warp has not produced), so the barrier is at most one phase
        // past PV_x's and a plain parity wait is exact -- no per-block bookkeeping.
        auto pv_done = [&](int x) {
            if (x >= 0) mbar_wait(o_done + (x & 1), (x >> 1) & 1);
        };
        constexpr int BB = B > 0 ? B : 64;
        const int bcols = B > 0 ? B : p.b;
        const float2 scl2 = make_float2(p.scale_log2, p.scale_log2);
        // output row of query block qb, token rr: block-major, or (unblockify fused) the token's
        // position in the latent
        auto orow_offset = [&](int u, int qb, int rr_) -> int64_t {
            const int64_t idx = (static_cast<int64_t>(u) * p.nqb + qb) * p.b + rr_;
            if (!p.lat) return idx * D;
            const int e = u / p.lg.heads, hd = u % p.lg.heads;
            const int nw = qb % p.lg.nw(), nh = (qb / p.lg.nw()) % p.lg.nh(), nt = qb / (p.lg.nw() * p.lg.nh());
            const int dw = rr_ % p.lg.bw, dh = (rr_ / p.lg.bw) % p.lg.bh, dt = rr_ / (p.lg.bw * p.lg.bh);
            const int64_t tok = ((static_cast<int64_t>(e) * p.lg.T + nt * p.lg.bt + dt) * p.lg.H + nh * p.lg.bh + dh) *
                                    p.lg.W + nw * p.lg.bw + dw;
            return (tok * p.lg.heads + hd) * D;
        };
        FragMeta pend[2];  // split-tile fragments of this CTA (stream-K tail: at most two)
        int npend = 0;
        int jg = 0;
        for (int f = 0; f < n_frag; ++f) {
            const int lb = f & 1;
            const uint8_t* list = lists + static_cast<size_t>(lb) * p.max_list * esz;
            mbar_wait(list_full + lb, (f >> 1) & 1);
            const FragMeta fm = meta[lb];
            const int nf = fm.e1 - fm.e0;
            const int tile = fm.tile, u = fm.u;
            const int qb = half ? fm.qb1 : fm.qb0;
            const bool valid = rr < p.b && qb >= 0;

            // ---------------------------------------------------------- online softmax
            float m = -INFINITY, l = 0.0f;
            const uint32_t list_s = smem_u32(list) + fm.e0 * esz;
            for (int idx = 0; idx < nf; ++idx) {
                const int j = jg + idx;
                const int buf = j & 1;
                if (threadIdx.x == 64) stamp(p, 4, j);  // softmax warp 2 lane 0: waiting for S_j
                mbar_wait(s_full + buf, (j >> 1) & 1);
                if (threadIdx.x == 64) stamp(p, 5, j);  // S_j seen
                if (threadIdx.x == 64 && j == 0) stamp_cta(p, 2);
                tc_fence_after();
                const uint32_t t_s = t_o + L::kSColBase + buf * 64;
                // rows of one warp all lie in one half -> visibility is warp-uniform
                const uint32_t ent = L16 ? ld_shared_u16(list_s + idx * 2) : ld_shared_u32(list_s + idx * 4);
                const bool vis = ((ent >> (mshift + half)) & 1) && (p.ablate & 1) == 0;
                if (vis) {
                    uint32_t pk[32];
                    float sv[64];
                    tmem_ld32(t_s, *reinterpret_cast<uint32_t(*)[32]>(sv));
                    tmem_ld32(t_s + 32, *reinterpret_cast<uint32_t(*)[32]>(sv + 32));
                    tmem_wait_ld();
                    if (threadIdx.x == 64) stamp(p, 7, j);  // S_j in registers
                    if (B == 0) {
#pragma unroll
                        for (int c = 0; c < 64; ++c)
                            if (c >= bcols) sv[c] = -INFINITY;  // generic block size
                    }
                    auto row_max = [&]() {
                        float mx4[4];
#pragma unroll
                        for (int q4 = 0; q4 < 4; ++q4) {
                            float a = -INFINITY;
#pragma unroll
                            for (int c = q4 * 16; c < q4 * 16 + 16; c += 2) {
                                if (c + 1 < BB) a = fmax3(a, sv[c], sv[c + 1]);
                                else if (c < BB) a = fmaxf(a, sv[c]);
                            }
                            mx4[q4] = a;
                        }
                        return fmaxf(fmaxf(mx4[0], mx4[1]), fmaxf(mx4[2], mx4[3])) * p.scale_log2;
                    };
                    // P_j = 2^(s * scale * log2e - m) packed to bf16 pairs; returns the block row sum
                    auto exps = [&]() {
                        const float bias = valid ? -m : -INFINITY;  // padding rows -> p = 0
                        const float2 bias2 = make_float2(bias, bias);
                        float2 acc[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f),
                                         make_float2(0.f, 0.f)};
#pragma unroll
                        for (int c2 = 0; c2 < 32; ++c2) {
                            const float2 x = __ffma2_rn(make_float2(sv[2 * c2], sv[2 * c2 + 1]), scl2, bias2);
                            float2 e;
                            if ((POLY >> c2) & 1u) {  // this column pair on the FMA pipe
                                e = exp2_poly2(x);
                                if (2 * c2 >= BB) e.x = 0.0f;
                                if (2 * c2 + 1 >= BB) e.y = 0.0f;
                            } else {
                                e.x = (2 * c2 < BB) ? exp2_approx(x.x) : 0.0f;
                                e.y = (2 * c2 + 1 < BB) ? exp2_approx(x.y) : 0.0f;
                            }
                            if (B == 0) {
                                if (2 * c2 >= bcols) e.x = 0.0f;
                                if (2 * c2 + 1 >= bcols) e.y = 0.0f;
                            }
                            if (2 * c2 < BB) acc[c2 & 3] = __fadd2_rn(acc[c2 & 3], e);
                            pk[c2] = pack_bf16x2(e.x, e.y);
                        }
                        const float2 s01 = __fadd2_rn(__fadd2_rn(acc[0], acc[1]), __fadd2_rn(acc[2], acc[3]));
                        return s01.x + s01.y;
                    };
                    // Running max without a per-block max: the row's first visible block sets m
                    // exactly (its O row is still zero); later blocks are exponentiated against the
                    // running m directly, and only a block whose row sum exceeds kOverflowSum (some
                    // score grew by ~10 in log2 units, or overflowed to inf) takes the exact path:
                    // true block max, O and l rescaled, P recomputed.  Values below that bound are
                    // exact-range fp32 / bf16, so the result is the usual online softmax.
                    if (__any_sync(0xffffffffu, valid && m == -INFINITY)) {
                        const float mx = row_max();
                        if (valid && m == -INFINITY) m = mx;
                    }
                    float lsum = exps();
                    if (threadIdx.x == 64) stamp(p, 8, j);  // exps done
                    const bool over = valid && lsum > kOverflowSum;
                    if (__any_sync(0xffffffffu, over)) {
                        const float m_new = over ? row_max() : m;
                        const float factor = over ? exp2_approx(m - m_new) : 1.0f;
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
                        m = m_new;
                        lsum = exps();
                    }
                    l += lsum;
                    if (threadIdx.x == 64) stamp(p, 9, j);  // P_j ready
                    tmem_st32(t_s, pk);
                } else {
                    uint32_t zero[32];
#pragma unroll
                    for (int c = 0; c < 32; ++c) zero[c] = 0u;
                    tmem_st32(t_s, zero);
                }
                tmem_wait_st();
                if (threadIdx.x == 64) stamp(p, 10, j);  // P_j stored
                tc_fence_before();
                if (threadIdx.x == 64) stamp(p, 6, j);  // about to arrive P_j
                __syncwarp();
                if (lane == 0) stamp(p, 9 + warp, j);  // per-warp arrival (warps 2-5 -> stamps 11-14)
                if (lane == 0) mbar_arrive(p_full + buf);
                // every o_done phase gets a waiter (compute-sanitizer synccheck): PV_{j-1} was issued
                // before S_{j+1}, which this warp waits for next, so this costs nothing
                pv_done(j - 1);
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(list_empty + lb);  // this warp is done with the list
            pv_done(jg + nf - 2);
            pv_done(jg + nf - 1);
            tc_fence_after();
            if (threadIdx.x == 64) stamp_cta(p, 3);

            // ---------------------------------------------------------- epilogue
            const int64_t orow_idx = (static_cast<int64_t>(u) * p.nqb + qb) * p.b + rr;
            if (fm.whole) {
                const int64_t orow_off = orow_offset(u, qb, rr);
                const float inv = l > 0.0f ? 1.0f / l : 0.0f;
                bf16* orow = p.o + orow_off;
#pragma unroll 1
                for (int c0 = 0; c0 < D; c0 += 32) {
                    uint32_t ov[32];
                    if (nf > 0) {
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
                    p.lse[orow_idx] = l > 0.0f ? (m + __log2f(l)) * 0.69314718055994531f : -INFINITY;
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(o_free);
            } else {
                // fragment of a split tile: unnormalised fp32 partial + (m, l)
                float* po = p.part_o + (static_cast<int64_t>(fm.slot) * 128 + r) * D;
#pragma unroll 1
                for (int c0 = 0; c0 < D; c0 += 32) {
                    uint32_t ov[32];
                    if (nf > 0) {
                        tmem_ld32(t_o + c0, ov);
                        tmem_wait_ld();
                    } else {
#pragma unroll
                        for (int c = 0; c < 32; ++c) ov[c] = 0u;
                    }
                    float4* dst = reinterpret_cast<float4*>(po + c0);
#pragma unroll
                    for (int c = 0; c < 8; ++c)
                        dst[c] = make_float4(__uint_as_float(ov[4 * c]), __uint_as_float(ov[4 * c + 1]),
                                             __uint_as_float(ov[4 * c + 2]), __uint_as_float(ov[4 * c + 3]));
                }
                float* pml = p.part_ml + static_cast<int64_t>(fm.slot) * 256;
                pml[r] = (nf > 0 && l > 0.0f) ? m : -INFINITY;
                pml[128 + r] = nf > 0 ? l : 0.0f;
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(o_free);
                __threadfence();
                if (t == 0) stamp_cta(p, 4);
                named_bar_sync(1, 128);
                if (t == 0) atomicAdd(p.counters + tile, 1);  // this fragment's partial is written
                pend[npend++] = fm;
            }
            jg += nf;
        }

        // ---------------------------------------------------------- split-tile merge
        // Every CTA holding a fragment of a split tile merges a slice of its 128 rows (fragment q of
        // nf takes rows [128 q / nf, 128 (q + 1) / nf)), in fragment order (deterministic), once it
        // has finished ALL its own fragments -- so no CTA waits while a partial of its own is
        // unwritten, and the co-resident grid cannot deadlock.  The K ring is idle by now (every
        // fragment's MMAs completed) and holds the per-row merge weights.  The tile counter counts
        // nf partial arrivals, then nf merge completions; the last merger re-zeroes it.
#ifdef PBSA_K3_TRACE
        if (t == 0 && p.trace != nullptr) p.trace[15 * 256 + 9 * 1024 + blockIdx.x] = jg;  // list entries processed
#endif
        // Q, K ring and V ring are idle by now (every fragment's loads were consumed by its MMAs):
        // the slice's partial rows are staged there by bulk copies (one per fragment, all in flight
        // together), the per-row weights after them
        constexpr uint32_t kStageBytes = L::kOffBar;                 // [0, kOffBar): Q + K + V rings
        float* stage = reinterpret_cast<float*>(smem);              // [nf][nrows][D] fp32
        float* wsm = stage + (128 + 8) * D;                         // [8][128] weights, [8 * 128 + r] 1 / sum,
        static_assert((128 + 8) * D * 4 + (9 * 128 + 8) * 4 <= kStageBytes, "merge staging");  // [9 * 128 + q] slots
        for (int i = 0; i < npend; ++i) {
            const FragMeta pm = pend[i];
            const int nfr = pm.nf < 8 ? pm.nf : 8;
            const int q = cta - pm.first_cta;
            const int r0 = q * 128 / nfr, nrows = (q + 1) * 128 / nfr - r0;
            int* sl = reinterpret_cast<int*>(wsm + 9 * 128);  // partial slot of fragment q2
            if (t < nfr) {
                const int c2 = pm.first_cta + t;
                const int first2 = p.tail_base + static_cast<int>(range_begin(c2, p.vtotal, p.tail_grid) / p.vlen);
                sl[t] = 2 * c2 + (pm.tile == first2 ? 0 : 1);
            }
            named_bar_sync(1, 128);
            if (t == 0) {
                while (ld_acquire_gpu(p.counters + pm.tile) < nfr) __nanosleep(32);
                stamp_cta(p, 5);
                fence_proxy_async_global();
                const uint32_t bytes = static_cast<uint32_t>(nrows) * D * 4;
                mbar_arrive_expect_tx(merge_bar, bytes * nfr);
                for (int q2 = 0; q2 < nfr; ++q2)
                    bulk_g2s(stage + q2 * nrows * D, p.part_o + (static_cast<int64_t>(sl[q2]) * 128 + r0) * D, bytes,
                             merge_bar);
            }
            named_bar_sync(1, 128);  // the tile's partials are complete (t == 0 acquired the counter)
            if (t < nrows) {
                const int row = r0 + t;
                float mf[8], lf[8];
                float M = -INFINITY;
                for (int q2 = 0; q2 < nfr; ++q2) {
                    mf[q2] = __ldcg(p.part_ml + static_cast<int64_t>(sl[q2]) * 256 + row);
                    lf[q2] = __ldcg(p.part_ml + static_cast<int64_t>(sl[q2]) * 256 + 128 + row);
                    M = fmaxf(M, mf[q2]);
                }
                float Ls = 0.0f;
                for (int q2 = 0; q2 < nfr; ++q2) {
                    mf[q2] = mf[q2] == -INFINITY ? 0.0f : exp2_approx(mf[q2] - M);
                    Ls += mf[q2] * lf[q2];
                }
                for (int q2 = 0; q2 < nfr; ++q2) wsm[q2 * 128 + t] = mf[q2];
                wsm[8 * 128 + t] = Ls > 0.0f ? 1.0f / Ls : 0.0f;
                const int qb2 = (row >> 6) ? pm.qb1 : pm.qb0, rr2 = row & 63;
                if (rr2 < p.b && qb2 >= 0 && p.lse != nullptr)
                    p.lse[(static_cast<int64_t>(pm.u) * p.nqb + qb2) * p.b + rr2] =
                        Ls > 0.0f ? (M + __log2f(Ls)) * 0.69314718055994531f : -INFINITY;
            }
            mbar_wait(merge_bar, i & 1);
            named_bar_sync(1, 128);
            // (row, float4 column) items: a warp covers one 512-byte row per step
            constexpr int C4 = D / 4;
            const int items = nrows * C4;
            for (int it = t; it < items; it += 128) {
                const int rl = it / C4, c4 = it % C4;
                float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
                for (int q2 = 0; q2 < nfr; ++q2) {  // fragment order
                    const float w = wsm[q2 * 128 + rl];
                    const float4 x = reinterpret_cast<const float4*>(stage + (q2 * nrows + rl) * D)[c4];
                    acc.x += w * x.x;
                    acc.y += w * x.y;
                    acc.z += w * x.z;
                    acc.w += w * x.w;
                }
                const int row = r0 + rl;
                const int qb2 = (row >> 6) ? pm.qb1 : pm.qb0, rr2 = row & 63;
                if (rr2 >= p.b || qb2 < 0) continue;
                const float inv = wsm[8 * 128 + rl];
                uint2 w2;
                w2.x = pack_bf16x2(acc.x * inv, acc.y * inv);
                w2.y = pack_bf16x2(acc.z * inv, acc.w * inv);
                *reinterpret_cast<uint2*>(p.o + orow_offset(pm.u, qb2, rr2) + c4 * 4) = w2;
            }
            named_bar_sync(1, 128);  // wsm is rewritten by the next merge
            if (t == 0) {
                if (atomicAdd(p.counters + pm.tile, 1) == 2 * nfr - 1) p.counters[pm.tile] = 0;  // next launch
                stamp_cta(p, 6);
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc<kTmemCols>(tmem);
    }
#ifdef PBSA_K3_TRACE
    if (threadIdx.x == 0 && p.trace != nullptr) {
        uint32_t smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        stamp_cta(p, 7);
        p.trace[15 * 256 + 8 * 1024 + blockIdx.x] = smid;
    }
#endif
    if (p.gangs > 0 && threadIdx.x == 0) {
        // the last CTA out re-zeroes the gang counters for the next launch (every producer has
        // passed its last barrier: a CTA only exits after its producer finished all units)
        __threadfence();
        if (atomicAdd(p.gang_ctr + kMaxGangs, 1) == static_cast<int>(gridDim.x) - 1) {
            for (int g = 0; g <= p.gangs; ++g) p.gang_ctr[g] = 0;  // (+ the extra gang's)
            p.gang_ctr[kMaxGangs] = 0;
            __threadfence();
        }
    }
}

template <int D, int NSK, int NSV, int B, uint32_t POLY, bool L16>
int launch_impl(const bf16* q, const bf16* kp, const bf16* vp, BsaParams p, cudaStream_t s) {
    using L = Layout<D, NSK, NSV>;
    alignas(64) CUtensorMap tq, tk, tv;
    if (int rc = encode_k3_maps(q, kp, vp, p, D, &tq, &tk, &tv)) return rc;
    const size_t smem = L::bytes(p.max_list, p.bm_words, L16 ? 2 : 4);
    if (smem > 227 * 1024)
        return set_error(PBSA_EUNSUPPORTED, "bsa_fwd: visible list too long for shared memory");
    if (int rc = ensure_smem(reinterpret_cast<const void*>(bsa_fwd_kernel<D, NSK, NSV, B, POLY, L16>), smem, "bsa_fwd"))
        return rc;
    // persistent grid = the CTAs that are actually co-resident: __launch_bounds__(kThreads, 2) keeps
    // registers at two CTAs per SM, so shared memory decides
    int per_sm = 2;
    {
        int dev = 0, sm_smem = 0, reserved = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sm_smem, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
        cudaDeviceGetAttribute(&reserved, cudaDevAttrReservedSharedMemoryPerBlock, dev);
        if (sm_smem > 0 && 2 * (smem + static_cast<size_t>(reserved)) > static_cast<size_t>(sm_smem)) per_sm = 1;
    }
    const int slots = per_sm * num_sms();
    plan_schedule(p, slots, D);
    record_plan(p, L16, per_sm, smem);
    if (p.grid <= 0) return 0;
    if (launch_pdl(bsa_fwd_kernel<D, NSK, NSV, B, POLY, L16>, dim3(p.grid), dim3(kThreads), smem, s, tq, tk, tv, p) !=
        cudaSuccess)
        return check_launch("bsa_fwd_kernel");
    return check_launch("bsa_fwd_kernel");
}

}  // namespace

pbsa_bsa_plan& last_bsa_plan() {
    static thread_local pbsa_bsa_plan plan{};
    return plan;
}

size_t bsa_fwd_workspace(int units, int nqb, int d) {
    const size_t slots = kRing * static_cast<size_t>(2 * num_sms());
    const size_t tiles = static_cast<size_t>(units) * ((nqb + 1) / 2);
    return slots * 128 * d * 4 + slots * 256 * 4 + tiles * 4 + (kMaxGangs + 1) * 4 + 256;
}

static long long* g_trace = nullptr;

}  // namespace pbsa

extern "C" void pbsa_debug_trace_buffer(void* p) { pbsa::g_trace = static_cast<long long*>(p); }

namespace pbsa {

int launch_bsa_fwd(const bf16* q, const bf16* k_pool, const bf16* v_pool, int n_slots,
                   const int32_t* dense, int dense_stride, int n_dense, const int32_t* local,
                   int local_stride, int n_local, const int32_t* sel, int k, int nqb, int b, int d,
                   int units, float scale, bf16* o, float* lse, void* ws, size_t ws_bytes, cudaStream_t s,
                   const LatentGeom* lat, int sel_rows, int sel_row0, const int32_t* tile_pairs) {
    BsaParams p{};
    p.pairs = tile_pairs;
    p.lat = lat != nullptr;
    if (lat) p.lg = *lat;
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
    p.sel_rows = sel_rows > 0 ? sel_rows : nqb;
    p.sel_row0 = sel_row0;
    p.k = (n_local > 0) ? k : 0;
    p.o = o;
    p.lse = lse;
    p.scale_log2 = scale * 1.4426950408889634f;
    {
        static const int ablate = getenv("PBSA_ABLATE") ? atoi(getenv("PBSA_ABLATE")) : 0;
        p.ablate = ablate;
        p.trace = g_trace;
    }
    p.bm_words = (n_local + 31) / 32 + 1;
    p.max_list = n_dense + (p.k > 0 ? (2 * p.k < n_local ? 2 * p.k : n_local) : 0);
    p.tiles_per_unit = (nqb + 1) / 2;
    p.n_tiles = units * p.tiles_per_unit;
    p.vlen = p.max_list > 0 ? p.max_list : 1;
    if (units == 0 || nqb == 0) return 0;
    if (ws != nullptr) {
        if (ws_bytes < bsa_fwd_workspace(units, nqb, d))
            return set_error(PBSA_EINVAL, "bsa_fwd: workspace too small");
        const size_t slots = kRing * static_cast<size_t>(2 * num_sms());
        p.part_o = static_cast<float*>(ws);
        p.part_ml = p.part_o + slots * 128 * d;
        p.counters = reinterpret_cast<int*>(p.part_ml + slots * 256);
        p.gang_ctr = p.counters + p.n_tiles;
    }
    // 16-bit visible-list entries only where 32-bit lists would cost the second CTA per SM (long
    // lists, e.g. config 5) and the pool is small enough to index with 14 bits
    const size_t smem32 = Layout<128, 2, 2>::bytes(p.max_list, p.bm_words, 4);
    const bool l16 = n_slots < 16384 && 2 * (smem32 + 1024) > 228 * 1024;
#define PBSA_K3(DD, NS, BB)                                                                       \
    return l16 ? launch_impl<DD, NS, NS, BB, kPolyMask, true>(q, k_pool, v_pool, p, s)            \
               : launch_impl<DD, NS, NS, BB, kPolyMask, false>(q, k_pool, v_pool, p, s)
    if (d == 128) {
        if (b == 60) PBSA_K3(128, 2, 60);
        if (b == 64) PBSA_K3(128, 2, 64);
        PBSA_K3(128, 2, 0);
    }
    if (b == 60) PBSA_K3(64, 3, 60);
    if (b == 64) PBSA_K3(64, 3, 64);
    PBSA_K3(64, 3, 0);
#undef PBSA_K3
}

}  // namespace pbsa
