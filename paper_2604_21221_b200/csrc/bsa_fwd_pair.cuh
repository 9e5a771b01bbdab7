// bsa_fwd_pair.cuh -- K3 variant over PAIRS of visible key blocks (included by bsa_fwd.cu).
//
// Same op, tile, list, schedule and outputs as bsa_fwd_kernel (see bsa_fwd.cu); what changes is how
// a CTA walks its tile's visible list:
//   * S for two consecutive list entries (a, b) is ONE tcgen05.mma per K-step at N = 128: K_a and
//     K_b are loaded into one 128-row pair slot, S_ab = Q [K_a; K_b]^T.  An SS M128 N64 MMA costs 48
//     cycles (operand-bandwidth bound, profiles/r01_umma_throughput.md), an N128 one 64: S costs 256
//     instead of 384 tensor cycles per key block.
//   * Two softmax warpgroups: WG A (warps 2-5) owns entry a of every pair, WG B (warps 6-9) entry b.
//     Each runs its own online softmax into its OWN accumulator (O_A, O_B in TMEM) with its own
//     running max and sum, so the groups never synchronise per block; the epilogue merges the two
//     (m, l, O) states row by row (the partner warp of the same TMEM lane quarter exchanges m and l
//     through shared memory once per tile).
//   * One CTA per SM: TMEM O_A [0, D), O_B [D, 2D), S pair buffers [256, 384) and [384, 512)
//     (P_a packed over the first 32 columns of its S half, P_b likewise), double-buffered so the S
//     of pair i+1 is computed while pair i is in the softmax.  Shared memory: Q (32 KB), a ring of
//     NKP 32 KB K pair slots, a ring of NSV 16 KB V slots, the double-buffered lists.
// A fragment with an odd number of entries gets one dummy entry (the fragment's first slot again,
// visible to neither half): its P is zero, so it contributes nothing.
// Roofline: tensor core; per key block the MMA needs 256 (S) + 256 (PV) cycles instead of 640.

template <int D, int NKP, int NSV>
struct PairLayout {
    static constexpr int kHalves = D / 64;
    static constexpr uint32_t kQBytes = kHalves * 128 * 128;   // [half][128 rows][128 B]
    static constexpr uint32_t kKPBytes = kHalves * 128 * 128;  // pair slot: [half][K_a 64 rows ++ K_b 64 rows][128 B]
    static constexpr uint32_t kVBytes = kHalves * 64 * 128;    // one V slot: [half][64 rows][128 B]
    static constexpr uint32_t kOffQ = 0;
    static constexpr uint32_t kOffK = kOffQ + kQBytes;
    static constexpr uint32_t kOffV = kOffK + NKP * kKPBytes;
    static constexpr uint32_t kOffBar = kOffV + NSV * kVBytes;
    // q_full, q_empty, kp_full/empty[NKP], v_full/empty[NSV], s_full[2], pa_full[2], pb_full[2],
    // oa_done[2], ob_done[2], o_free, list_full[2], list_empty[2], merge
    static constexpr int kNumBars = 2 + 2 * NKP + 2 * NSV + 10 + 1 + 4 + 1;
    static constexpr uint32_t kOffMeta = kOffBar + kNumBars * 8;
    static constexpr uint32_t kOffMisc = kOffMeta + 2 * sizeof(FragMeta);
    static constexpr uint32_t kOffXch = kOffMisc + 16;  // [m, l][128 rows] per group: 2 x 2 x 128 f32
    static constexpr uint32_t kOffList = kOffXch + 2 * 2 * 128 * 4;
    static constexpr uint32_t kOA = 0, kOB = D, kSBase = 256;  // TMEM columns
    static size_t bytes(int max_list, int bm_words, int entry_bytes) {
        const size_t lb = (2 * static_cast<size_t>(max_list) * entry_bytes + 15) & ~size_t(15);
        return 1024 + kOffList + lb + 2 * static_cast<size_t>(bm_words) * 4;
    }
};

constexpr int kPairThreads = 320;  // producer, MMA issuer, two softmax warpgroups

template <int D, int NKP, int NSV, int B, uint32_t POLY, bool L16>
__global__ void __launch_bounds__(kPairThreads, 1)
    bsa_fwd_pair_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                        const __grid_constant__ CUtensorMap tm_v, const BsaParams p) {
    using L = PairLayout<D, NKP, NSV>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* q_smem = smem + L::kOffQ;
    uint8_t* k_smem = smem + L::kOffK;
    uint8_t* v_smem = smem + L::kOffV;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::kOffBar);
    uint64_t* q_full = bars;
    uint64_t* q_empty = bars + 1;
    uint64_t* kp_full = bars + 2;
    uint64_t* kp_empty = kp_full + NKP;
    uint64_t* v_full = kp_empty + NKP;
    uint64_t* v_empty = v_full + NSV;
    uint64_t* s_full = v_empty + NSV;
    uint64_t* pa_full = s_full + 2;
    uint64_t* pb_full = pa_full + 2;
    uint64_t* oa_done = pb_full + 2;
    uint64_t* ob_done = oa_done + 2;
    uint64_t* o_free = ob_done + 2;
    uint64_t* list_full = o_free + 1;
    uint64_t* list_empty = list_full + 2;
    uint64_t* merge_bar = list_empty + 2;
    FragMeta* meta = reinterpret_cast<FragMeta*>(smem + L::kOffMeta);
    uint32_t* misc = reinterpret_cast<uint32_t*>(smem + L::kOffMisc);
    float* xch = reinterpret_cast<float*>(smem + L::kOffXch);
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
        for (int s = 0; s < NKP; ++s) {
            mbar_init(kp_full + s, 1);
            mbar_init(kp_empty + s, 1);
        }
        for (int s = 0; s < NSV; ++s) {
            mbar_init(v_full + s, 1);
            mbar_init(v_empty + s, 1);
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init(s_full + s, 1);
            mbar_init(pa_full + s, 4);  // one elected arrival per warp of the group
            mbar_init(pb_full + s, 4);
            mbar_init(oa_done + s, 1);
            mbar_init(ob_done + s, 1);
            mbar_init(list_full + s, 1);
            mbar_init(list_empty + s, 9);  // MMA warp + 8 softmax warps
        }
        mbar_init(o_free, 8);
        mbar_init(merge_bar, 1);
        fence_barrier_init();
        tma_prefetch(&tm_q);
        tma_prefetch(&tm_k);
        tma_prefetch(&tm_v);
    }
    if (warp == 1) tmem_alloc<512>(misc);
    if (warp >= 2) {
        // zero the rows >= b of the Q tile halves and of every K pair / V ring slot once: TMA only
        // ever writes the b valid rows (S stays finite; P V exact)
        const int t = threadIdx.x - 64;
        for (int e = t; e < 128 * L::kHalves * 8; e += 256) {
            const int chunk = e & 7, rh = e >> 3;
            const int h = rh % L::kHalves, row = rh / L::kHalves;
            if ((row & 63) >= p.b)
                *reinterpret_cast<uint4*>(q_smem + h * 16384 + row * 128 + chunk * 16) = make_uint4(0, 0, 0, 0);
        }
        // K pair slots and V slots as 64-row boxes of 8 KB: (NKP * 2 + NSV) * kHalves of them
        for (int e = t; e < (2 * NKP + NSV) * L::kHalves * 64 * 8; e += 256) {
            const int chunk = e & 7, row = (e >> 3) & 63, bx = e >> 9;
            if (row >= p.b)
                *reinterpret_cast<uint4*>(k_smem + bx * 8192 + row * 128 + chunk * 16) = make_uint4(0, 0, 0, 0);
        }
        fence_proxy_async_smem();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = misc[0];
    pdl_wait();  // the preceding kernels' outputs (selections, Q, the ingest) are visible from here
    if (threadIdx.x == 0) stamp_cta(p, 0);

    if (warp == 0) {
        // ============================================================== TMA producer + lists
        const uint32_t kv_tx = static_cast<uint32_t>(L::kHalves) * static_cast<uint32_t>(p.b) * 128u;
        int pgj = 0, q_uses = 0;  // pairs issued so far, Q tiles loaded
        for (int f = 0; f < n_frag; ++f) {
            const int lb = f & 1;
            mbar_wait(list_empty + lb, ((f >> 1) & 1) ^ 1);
            uint8_t* list = lists + static_cast<size_t>(lb) * p.max_list * esz;
            const FragPlan fp = plan_fragment(p, cta, f);
            gang_wait(p, cta, f);
            const int run = build_visible_list<L16>(p, fp, list, bm);
            const FragMeta fm = make_meta(p, fp, run);
            if (lane == 0) meta[lb] = fm;
            if (lane == 0 && f == 0) stamp_cta(p, 1);
            __syncwarp();
            if (lane == 0) mbar_arrive(list_full + lb);
            const int nf = fm.e1 - fm.e0;
            const int np = (nf + 1) >> 1;
            if (nf > 0) {
                if (q_uses > 0) mbar_wait(q_empty, (q_uses - 1) & 1);
                const uint32_t qbytes = (fm.has2 ? 2u : 1u) * L::kHalves * static_cast<uint32_t>(p.b) * 128u;
                if (elect_one()) {
                    mbar_arrive_expect_tx(q_full, qbytes);
                    for (int r = 0; r < (fm.has2 ? 2 : 1); ++r)
                        for (int h = 0; h < L::kHalves; ++h) {
                            if (p.lat) {
                                const int qb = fm.qb0 + r, e = fm.u / p.lg.heads, hd = fm.u % p.lg.heads;
                                const int nw = qb % p.lg.nw(), nh = (qb / p.lg.nw()) % p.lg.nh();
                                const int nt = qb / (p.lg.nw() * p.lg.nh());
                                tma_load_5d(q_smem + h * 16384 + r * 8192, &tm_q, q_full, hd * D + h * 64,
                                            nw * p.lg.bw, nh * p.lg.bh, nt * p.lg.bt, e);
                            } else {
                                tma_load_3d(q_smem + h * 16384 + r * 8192, &tm_q, q_full, h * 64, 0,
                                            fm.u * p.nqb + fm.qb0 + r);
                            }
                        }
                }
                __syncwarp();
                ++q_uses;
                // entry 2i + x of the fragment (x = 0: a, 1: b); the odd tail's b is entry 0 again
                auto pool_row = [&](int idx) -> int {
                    const int e = idx < nf ? idx : 0;
                    return (fm.u * p.n_slots + list_slot<L16>(list, fm.e0 + e)) * 64;
                };
                auto load_v = [&](int i) {  // V_a and V_b of pair i
#pragma unroll 1
                    for (int x = 0; x < 2; ++x) {
                        const int j = 2 * (pgj + i) + x;
                        const int s = j % NSV;
                        mbar_wait(v_empty + s, ((j / NSV) & 1) ^ 1);
                        const int row0 = pool_row(2 * i + x);
                        if (elect_one()) {
                            if (p.ablate & 2) {
                                mbar_arrive(v_full + s);
                            } else {
                                mbar_arrive_expect_tx(v_full + s, kv_tx);
                                for (int h = 0; h < L::kHalves; ++h)
                                    tma_load_2d(v_smem + s * L::kVBytes + h * 8192, &tm_v, v_full + s, h * 64, row0);
                            }
                        }
                        __syncwarp();
                    }
                };
                for (int i = 0; i < np; ++i) {
                    const int pg = pgj + i;
                    const int s = pg % NKP;
                    mbar_wait(kp_empty + s, ((pg / NKP) & 1) ^ 1);
                    const int ra = pool_row(2 * i), rb = pool_row(2 * i + 1);
                    if (elect_one()) {
                        if (p.ablate & 2) {
                            mbar_arrive(kp_full + s);
                        } else {
                            mbar_arrive_expect_tx(kp_full + s, 2 * kv_tx);
                            for (int h = 0; h < L::kHalves; ++h) {
                                uint8_t* dst = k_smem + s * L::kKPBytes + h * 16384;
                                tma_load_2d(dst, &tm_k, kp_full + s, h * 64, ra);
                                tma_load_2d(dst + 8192, &tm_k, kp_full + s, h * 64, rb);
                            }
                        }
                    }
                    __syncwarp();
                    if (i >= 1) load_v(i - 1);
                }
                load_v(np - 1);
                pgj += np;
            }
            gang_arrive(p, cta);
        }
    } else if (warp == 1) {
        // ============================================================== tcgen05 issuer
        constexpr uint32_t idesc_s = idesc_bf16_f32(128, 128, 0, 0);
        constexpr uint32_t idesc_o = idesc_bf16_f32(128, D, 0, 1);
        const bool do_mma = (p.ablate & 4) == 0;
        const uint64_t qdesc = smem_desc_sw128(smem_u32(q_smem), 16, 1024);
        const uint64_t kdesc = smem_desc_sw128(smem_u32(k_smem), 16, 1024);
        const uint64_t vdesc = smem_desc_sw128(smem_u32(v_smem), 8192, 1024);
        int pgj = 0, q_uses = 0;
        auto issue_s = [&](int pg) {
            const int s = pg % NKP;
            mbar_wait(kp_full + s, (pg / NKP) & 1);
            tc_fence_after();
            const uint32_t d_tmem = tmem + L::kSBase + (pg & 1) * 128;
            const uint64_t kd = kdesc + ((s * L::kKPBytes) >> 4);
            if (elect_one()) {
                if (do_mma) {
#pragma unroll
                    for (int kk = 0; kk < D / 16; ++kk) {
                        const uint32_t off = ((kk >> 2) * 16384 + (kk & 3) * 32) >> 4;
                        mma_ss(d_tmem, qdesc + off, kd + off, idesc_s, kk > 0 ? 1u : 0u);
                    }
                }
                mma_commit(kp_empty + s);
                mma_commit(s_full + (pg & 1));
            }
            __syncwarp();
        };
        auto issue_pv = [&](int pg, int x, bool first) {  // O_x += P_x V_x of pair pg
            uint64_t* pf = x == 0 ? pa_full : pb_full;
            mbar_wait(pf + (pg & 1), (pg >> 1) & 1);
            stamp(p, x == 0 ? 2 : 11, pg);  // MMA: P_x seen
            const int j = 2 * pg + x;
            const int sv = j % NSV;
            mbar_wait(v_full + sv, (j / NSV) & 1);
            tc_fence_after();
            const uint32_t a_tmem = tmem + L::kSBase + (pg & 1) * 128 + x * 64;
            const uint64_t vd = vdesc + ((sv * L::kVBytes) >> 4);
            if (elect_one()) {
                if (do_mma) {
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk)
                        mma_ts(tmem + (x == 0 ? L::kOA : L::kOB), a_tmem + kk * 8, vd + ((kk * 2048) >> 4), idesc_o,
                               (!first || kk > 0) ? 1u : 0u);
                }
                mma_commit(v_empty + sv);
                mma_commit((x == 0 ? oa_done : ob_done) + (pg & 1));
            }
            __syncwarp();
            stamp(p, x == 0 ? 3 : 12, pg);  // MMA: PV_x issued
        };
        for (int f = 0; f < n_frag; ++f) {
            const int lb = f & 1;
            mbar_wait(list_full + lb, (f >> 1) & 1);
            const int nf = meta[lb].e1 - meta[lb].e0;
            const int np = (nf + 1) >> 1;
            __syncwarp();
            if (lane == 0) mbar_arrive(list_empty + lb);
            if (f > 0) mbar_wait(o_free, (f - 1) & 1);  // the previous epilogue has read O_A / O_B
            if (nf == 0) continue;
            mbar_wait(q_full, q_uses & 1);
            tc_fence_after();
            issue_s(pgj);
            for (int i = 0; i < np; ++i) {
                const int pg = pgj + i;
                stamp(p, 0, pg);  // MMA: before issuing S_{pg+1}
                if (i + 1 < np) issue_s(pg + 1);
                stamp(p, 1, pg);  // MMA: S_{pg+1} issued
                issue_pv(pg, 0, i == 0);
                issue_pv(pg, 1, i == 0);
            }
            if (elect_one()) mma_commit(q_empty);
            __syncwarp();
            ++q_uses;
            pgj += np;
        }
    } else {
        // ============================================================== softmax groups
        const int t = threadIdx.x - 64;      // 0 .. 255
        const int grp = (warp - 2) >> 2;      // 0: entry a of every pair (O_A), 1: entry b (O_B)
        const int quarter = warp & 3;
        const int r = quarter * 32 + lane;
        const int half = r >> 6, rr = r & 63;
        const uint32_t lane_base = static_cast<uint32_t>(quarter * 32) << 16;
        const uint32_t t_row = tmem + lane_base;
        const uint32_t t_my_o = t_row + (grp == 0 ? L::kOA : L::kOB);
        uint64_t* my_p_full = grp == 0 ? pa_full : pb_full;
        uint64_t* my_o_done = grp == 0 ? oa_done : ob_done;
        // wait until this group's PV of pair x has completed (x is the latest of its parity that can
        // have been issued: PV_{x+2} needs this group's P_{x+2}) -- a plain parity wait is exact
        auto pv_done = [&](uint64_t* done, int x) {
            if (x >= 0) mbar_wait(done + (x & 1), (x >> 1) & 1);
        };
        constexpr int BB = B > 0 ? B : 64;
        const int bcols = B > 0 ? B : p.b;
        const float2 scl2 = make_float2(p.scale_log2, p.scale_log2);
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
        FragMeta pend[2];
        int npend = 0;
        int pgj = 0;
        for (int f = 0; f < n_frag; ++f) {
            const int lb = f & 1;
            const uint8_t* list = lists + static_cast<size_t>(lb) * p.max_list * esz;
            mbar_wait(list_full + lb, (f >> 1) & 1);
            const FragMeta fm = meta[lb];
            const int nf = fm.e1 - fm.e0;
            const int np = (nf + 1) >> 1;
            const int tile = fm.tile, u = fm.u, qb0 = fm.qb0;
            const int qb = qb0 + half;
            const bool valid = rr < p.b && qb < p.nqb;

            // ---------------------------------------------------------- online softmax (own O)
            float m = -INFINITY, l = 0.0f;
            const uint32_t list_s = smem_u32(list) + fm.e0 * esz;
            for (int i = 0; i < np; ++i) {
                const int pg = pgj + i;
                const int buf = pg & 1;
                const int idx = 2 * i + grp;
                if (threadIdx.x == 64) stamp(p, 4, pg);   // group A warp 2: waiting for S
                if (threadIdx.x == 192) stamp(p, 7, pg);  // group B warp 6
                mbar_wait(s_full + buf, (pg >> 1) & 1);
                if (threadIdx.x == 64) stamp(p, 5, pg);
                if (threadIdx.x == 192) stamp(p, 8, pg);
                if (threadIdx.x == 64 && pg == 0) stamp_cta(p, 2);
                tc_fence_after();
                const uint32_t t_s = t_row + L::kSBase + buf * 128 + grp * 64;
                uint32_t ent = 0;
                if (idx < nf) ent = L16 ? ld_shared_u16(list_s + idx * 2) : ld_shared_u32(list_s + idx * 4);
                const bool vis = idx < nf && ((ent >> (mshift + half)) & 1) && (p.ablate & 1) == 0;
                if (vis) {
                    uint32_t pk[32];
                    float sv[64];
                    tmem_ld32(t_s, *reinterpret_cast<uint32_t(*)[32]>(sv));
                    tmem_ld32(t_s + 32, *reinterpret_cast<uint32_t(*)[32]>(sv + 32));
                    tmem_wait_ld();
                    if (B == 0) {
#pragma unroll
                        for (int c = 0; c < 64; ++c)
                            if (c >= bcols) sv[c] = -INFINITY;
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
                    auto exps = [&]() {
                        const float bias = valid ? -m : -INFINITY;
                        const float2 bias2 = make_float2(bias, bias);
                        float2 acc[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f),
                                         make_float2(0.f, 0.f)};
#pragma unroll
                        for (int c2 = 0; c2 < 32; ++c2) {
                            const float2 x = __ffma2_rn(make_float2(sv[2 * c2], sv[2 * c2 + 1]), scl2, bias2);
                            float2 e;
                            if ((POLY >> c2) & 1u) {  // this column pair on the FMA pipe (MUFU relief)
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
                    // the group's first visible block sets its running max exactly; later blocks
                    // exponentiate against it and only an overflowing row sum takes the exact path
                    if (__any_sync(0xffffffffu, valid && m == -INFINITY)) {
                        const float mx = row_max();
                        if (valid && m == -INFINITY) m = mx;
                    }
                    float lsum = exps();
                    const bool over = valid && lsum > kOverflowSum;
                    if (__any_sync(0xffffffffu, over)) {
                        const float m_new = over ? row_max() : m;
                        const float factor = over ? exp2_approx(m - m_new) : 1.0f;
                        pv_done(my_o_done, pg - 1);
                        tc_fence_after();
#pragma unroll 1
                        for (int c0 = 0; c0 < D; c0 += 32) {
                            uint32_t ov[32];
                            tmem_ld32(t_my_o + c0, ov);
                            tmem_wait_ld();
#pragma unroll
                            for (int c = 0; c < 32; ++c) ov[c] = __float_as_uint(__uint_as_float(ov[c]) * factor);
                            tmem_st32(t_my_o + c0, ov);
                        }
                        l *= factor;
                        m = m_new;
                        lsum = exps();
                    }
                    l += lsum;
                    tmem_st32(t_s, pk);
                } else {
                    uint32_t zero[32];
#pragma unroll
                    for (int c = 0; c < 32; ++c) zero[c] = 0u;
                    tmem_st32(t_s, zero);
                }
                tmem_wait_st();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(my_p_full + buf);
                if (threadIdx.x == 64) stamp(p, 6, pg);
                if (threadIdx.x == 192) stamp(p, 9, pg);
                if (lane == 0 && warp != 2 && warp != 6) stamp(p, 13, pg);  // (last writer wins: some other warp)
                pv_done(my_o_done, pg - 1);  // every phase gets a waiter; free (issued before S_{pg+1})
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(list_empty + lb);
            // both groups' PVs of the fragment complete (the epilogue reads O_A and O_B)
            pv_done(oa_done, pgj + np - 2);
            pv_done(oa_done, pgj + np - 1);
            pv_done(ob_done, pgj + np - 2);
            pv_done(ob_done, pgj + np - 1);
            tc_fence_after();
            if (threadIdx.x == 64) stamp_cta(p, 3);

            // ---------------------------------------------------------- merge the two states
            xch[(grp * 2 + 0) * 128 + r] = m;
            xch[(grp * 2 + 1) * 128 + r] = l;
            named_bar_sync(2 + quarter, 64);  // this quarter's warp of each group
            const float m_o = xch[((grp ^ 1) * 2 + 0) * 128 + r];
            const float l_o = xch[((grp ^ 1) * 2 + 1) * 128 + r];
            const float ma = grp == 0 ? m : m_o, mb = grp == 0 ? m_o : m;
            const float la = grp == 0 ? l : l_o, lb2 = grp == 0 ? l_o : l;
            const float M = fmaxf(ma, mb);
            const float wa = ma == -INFINITY ? 0.0f : exp2_approx(ma - M);
            const float wb = mb == -INFINITY ? 0.0f : exp2_approx(mb - M);
            const float Ls = la * wa + lb2 * wb;
            named_bar_sync(2 + quarter, 64);  // xch is rewritten by the next fragment

            // ---------------------------------------------------------- epilogue: this group's column half
            const int64_t orow_idx = (static_cast<int64_t>(u) * p.nqb + qb) * p.b + rr;
            const int c_lo = grp * (D / 2), c_hi = c_lo + D / 2;
            if (fm.whole) {
                const float inv = Ls > 0.0f ? 1.0f / Ls : 0.0f;
                bf16* orow = p.o + orow_offset(u, qb, rr);
#pragma unroll 1
                for (int c0 = c_lo; c0 < c_hi; c0 += 32) {
                    uint32_t oa[32], ob[32];
                    if (nf > 0) {
                        tmem_ld32(t_row + L::kOA + c0, oa);
                        tmem_ld32(t_row + L::kOB + c0, ob);
                        tmem_wait_ld();
                    } else {
#pragma unroll
                        for (int c = 0; c < 32; ++c) oa[c] = ob[c] = 0u;
                    }
                    if (valid) {
                        const float sa = wa * inv, sb = wb * inv;
                        uint4 pkd[4];
                        uint32_t* w = reinterpret_cast<uint32_t*>(pkd);
#pragma unroll
                        for (int c = 0; c < 16; ++c)
                            w[c] = pack_bf16x2(__uint_as_float(oa[2 * c]) * sa + __uint_as_float(ob[2 * c]) * sb,
                                               __uint_as_float(oa[2 * c + 1]) * sa + __uint_as_float(ob[2 * c + 1]) * sb);
                        uint4* dst = reinterpret_cast<uint4*>(orow + c0);
#pragma unroll
                        for (int c = 0; c < 4; ++c) dst[c] = pkd[c];
                    }
                }
                if (grp == 0 && valid && p.lse != nullptr)
                    p.lse[orow_idx] = Ls > 0.0f ? (M + __log2f(Ls)) * 0.69314718055994531f : -INFINITY;
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(o_free);
            } else {
                // fragment of a split tile: unnormalised fp32 partial (scaled to M) + (M, L)
                float* po = p.part_o + (static_cast<int64_t>(fm.slot) * 128 + r) * D;
#pragma unroll 1
                for (int c0 = c_lo; c0 < c_hi; c0 += 32) {
                    uint32_t oa[32], ob[32];
                    if (nf > 0) {
                        tmem_ld32(t_row + L::kOA + c0, oa);
                        tmem_ld32(t_row + L::kOB + c0, ob);
                        tmem_wait_ld();
                    } else {
#pragma unroll
                        for (int c = 0; c < 32; ++c) oa[c] = ob[c] = 0u;
                    }
                    float4* dst = reinterpret_cast<float4*>(po + c0);
#pragma unroll
                    for (int c = 0; c < 8; ++c)
                        dst[c] = make_float4(__uint_as_float(oa[4 * c]) * wa + __uint_as_float(ob[4 * c]) * wb,
                                             __uint_as_float(oa[4 * c + 1]) * wa + __uint_as_float(ob[4 * c + 1]) * wb,
                                             __uint_as_float(oa[4 * c + 2]) * wa + __uint_as_float(ob[4 * c + 2]) * wb,
                                             __uint_as_float(oa[4 * c + 3]) * wa + __uint_as_float(ob[4 * c + 3]) * wb);
                }
                if (grp == 0) {
                    float* pml = p.part_ml + static_cast<int64_t>(fm.slot) * 256;
                    pml[r] = (nf > 0 && Ls > 0.0f) ? M : -INFINITY;
                    pml[128 + r] = nf > 0 ? Ls : 0.0f;
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(o_free);
                __threadfence();
                if (t == 0) stamp_cta(p, 4);
                named_bar_sync(1, 256);
                if (t == 0) atomicAdd(p.counters + tile, 1);  // this fragment's partial is written
                pend[npend++] = fm;
            }
            pgj += np;
        }

        // ---------------------------------------------------------- split-tile merge (group A only)
        // identical to bsa_fwd_kernel's: every CTA holding a fragment of a split tile merges its slice
        // of the tile's rows in fragment order once all its own fragments are done; the Q / K / V
        // rings are idle and stage the partial rows
        float* stage = reinterpret_cast<float*>(smem);
        float* wsm = stage + (128 + 8) * D;
        static_assert((128 + 8) * D * 4 + (9 * 128 + 8) * 4 <= L::kOffBar, "merge staging");
        for (int i = 0; i < (t < 128 ? npend : 0); ++i) {
            const FragMeta pm = pend[i];
            const int nfr = pm.nf < 8 ? pm.nf : 8;
            const int q = cta - pm.first_cta;
            const int r0 = q * 128 / nfr, nrows = (q + 1) * 128 / nfr - r0;
            int* sl = reinterpret_cast<int*>(wsm + 9 * 128);
            if (t < nfr) {
                const int c2 = pm.first_cta + t;
                const int first2 = p.tail_base + static_cast<int>(range_begin(c2, p.vtotal, p.tail_grid) / p.vlen);
                sl[t] = 2 * c2 + (pm.tile == first2 ? 0 : 1);
            }
            named_bar_sync(6, 128);
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
            named_bar_sync(6, 128);
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
                const int qb2 = pm.qb0 + (row >> 6), rr2 = row & 63;
                if (rr2 < p.b && qb2 < p.nqb && p.lse != nullptr)
                    p.lse[(static_cast<int64_t>(pm.u) * p.nqb + qb2) * p.b + rr2] =
                        Ls > 0.0f ? (M + __log2f(Ls)) * 0.69314718055994531f : -INFINITY;
            }
            mbar_wait(merge_bar, i & 1);
            named_bar_sync(6, 128);
            constexpr int C4 = D / 4;
            const int items = nrows * C4;
            for (int it = t; it < items; it += 128) {
                const int rl = it / C4, c4 = it % C4;
                float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
                for (int q2 = 0; q2 < nfr; ++q2) {
                    const float w = wsm[q2 * 128 + rl];
                    const float4 x = reinterpret_cast<const float4*>(stage + (q2 * nrows + rl) * D)[c4];
                    acc.x += w * x.x;
                    acc.y += w * x.y;
                    acc.z += w * x.z;
                    acc.w += w * x.w;
                }
                const int row = r0 + rl;
                const int qb2 = pm.qb0 + (row >> 6), rr2 = row & 63;
                if (rr2 >= p.b || qb2 >= p.nqb) continue;
                const float inv = wsm[8 * 128 + rl];
                uint2 w2;
                w2.x = pack_bf16x2(acc.x * inv, acc.y * inv);
                w2.y = pack_bf16x2(acc.z * inv, acc.w * inv);
                *reinterpret_cast<uint2*>(p.o + orow_offset(pm.u, qb2, rr2) + c4 * 4) = w2;
            }
            named_bar_sync(6, 128);
            if (t == 0) {
                if (atomicAdd(p.counters + pm.tile, 1) == 2 * nfr - 1) p.counters[pm.tile] = 0;
                stamp_cta(p, 6);
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc<512>(tmem);
    }
    if (p.gangs > 0 && threadIdx.x == 0) {
        __threadfence();
        if (atomicAdd(p.gang_ctr + kMaxGangs, 1) == static_cast<int>(gridDim.x) - 1) {
            for (int g = 0; g < p.gangs; ++g) p.gang_ctr[g] = 0;
            p.gang_ctr[kMaxGangs] = 0;
            __threadfence();
        }
    }
}

template <int D, int NKP, int NSV, int B, uint32_t POLY, bool L16>
int launch_pair_impl(const bf16* q, const bf16* kp, const bf16* vp, BsaParams p, cudaStream_t s) {
    using L = PairLayout<D, NKP, NSV>;
    alignas(64) CUtensorMap tq, tk, tv;
    if (int rc = encode_k3_maps(q, kp, vp, p, D, &tq, &tk, &tv)) return rc;
    const size_t smem = L::bytes(p.max_list, p.bm_words, L16 ? 2 : 4);
    if (smem > 227 * 1024)
        return set_error(PBSA_EUNSUPPORTED, "bsa_fwd: visible list too long for shared memory");
    if (int rc = ensure_smem(reinterpret_cast<const void*>(bsa_fwd_pair_kernel<D, NKP, NSV, B, POLY, L16>), smem, "bsa_fwd_pair"))
        return rc;
    plan_schedule(p, num_sms(), D);  // one CTA (one tile in flight) per SM
    record_plan(p, L16, 1, smem);
    if (p.grid <= 0) return 0;
    if (launch_pdl(bsa_fwd_pair_kernel<D, NKP, NSV, B, POLY, L16>, dim3(p.grid), dim3(kPairThreads), smem, s, tq, tk, tv,
                   p) != cudaSuccess)
        return check_launch("bsa_fwd_pair_kernel");
    return check_launch("bsa_fwd_pair_kernel");
}
